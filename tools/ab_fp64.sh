# fp64 pull variants at c2: tools/ab_fp64.sh "ENV..." ...
for cfg in "$@"; do
  env $cfg python bench.py --no-cpu --no-fp64 --dtype fp64 --steps 3 --warmup 3 > gpurun_out/bench_f.json 2>gpurun_out/bench_f.err || tail -2 gpurun_out/bench_f.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_f.json')); r=d['roofline']
print('$cfg', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3])"
done
