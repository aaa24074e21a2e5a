# parity + A/B of the speculative push (K1 folded into K1a) at c2
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
for cfg in "1 1,4" "1 1,3" "1 2,2" "0 1,4"; do
  set -- $cfg
  BH_SPEC_PUSH=$1 BH_ELEM_COMBINE=$2 python bench.py --no-cpu --no-fp64 --steps 5 --warmup 3 > gpurun_out/bench_s.json 2>gpurun_out/bench_s.err || tail -3 gpurun_out/bench_s.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_s.json')); r=d['roofline']
print('spec=$1 comb=$2', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3], d['gpu_launches'])"
done
