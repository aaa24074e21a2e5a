# A/B of engine variants at c2 (fp32): python bench.py per environment setting
for cfg in "$@"; do
  env $cfg python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "$cfg" $(python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);r=d['roofline'];b=r['breakdown_ms_per_step'];print(round(d['value']),round(d['e2e']['value']),round(d['fp64']['value']),round(b['ms_vpull'],2),round(b['ms_upull'],2),round(b['ms_prep'],2),round(b['ms_control'],2),r['timed_step_ms'],r['timed_step_rounds'],r['profiled_step_ms'],d['clocks'])")
done
