# A/B of the elementwise kernel configs (UNR,MINB) at c2
for cfg in "1,4 1,4" "1,5 1,5" "1,6 1,6" "2,4 2,4" "1,5 1,4" "1,4 1,5"; do
  set -- $cfg
  BH_ELEM_PUSH=$1 BH_ELEM_COMBINE=$2 python bench.py --no-cpu ${ELEM_ARGS:---no-fp64} --steps 5 --warmup 3 > gpurun_out/bench_e.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_e.json')); r=d['roofline']
print('push=$1 comb=$2', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3], d['fp64'] and round(d['fp64']['value'],1))"
done
