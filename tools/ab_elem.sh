# A/B of the elementwise kernel configs (BH_ELEM_PUSH / BH_ELEM_COMBINE = "UNR,MINB", "p" = pipelined) at c2
for cfg in "${@:-1,4 1,4}"; do
  set -- $cfg
  BH_ELEM_PUSH=$1 BH_ELEM_COMBINE=$2 python bench.py --no-cpu ${ELEM_ARGS:---no-fp64} --steps 5 --warmup 3 > gpurun_out/bench_e.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_e.json')); r=d['roofline']
print('push=$1 comb=$2', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3])"
done
