python -m pytest tests/test_gpu_parity.py -q -x -k "variant" > gpurun_out/pytest_var.txt 2>&1; tail -2 gpurun_out/pytest_var.txt
for h in 0 3 1 2; do
  BH_PULL_HALF=$h python bench.py --no-cpu --no-fp64 --steps 5 --warmup 3 > gpurun_out/bench_h$h.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_h$h.json')); r=d['roofline']
print('half=$h', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'])"
done
