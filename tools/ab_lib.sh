# A/B of in-tree library builds (BH_LIBBHPP) at c2: tools/ab_lib.sh libA.so libB.so ...
for lib in "" "$@"; do
  BH_LIBBHPP=${lib:-paper_2312_06724_b200/_lib/libbhpp.so} python bench.py --no-cpu --no-fp64 --steps 5 --warmup 3 > gpurun_out/bench_l.json 2>gpurun_out/bench_l.err || tail -3 gpurun_out/bench_l.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_l.json')); r=d['roofline']
print('${lib:-default}', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3])"
done
