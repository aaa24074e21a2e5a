# Step-time jitter check: timed steps with and without the device start gate.
for i in 1 2 3; do
 for cfg in "BH_BENCH_NO_GATE=1" "X=gate"; do
  env $cfg python bench.py --steps 10 --warmup 3 --no-cpu --no-fp64 > gpurun_out/j.json 2>gpurun_out/j.err
  echo "$cfg" $(python -c "import json;d=json.loads(open('gpurun_out/j.json').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['value']),round(d['e2e']['value']),r['timed_step_ms'])")
 done
done
