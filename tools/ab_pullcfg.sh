# A/B of k_pull_sw geometry (S rows in flight, blocks/SM) per side at c2: tools/ab_pullcfg.sh "V U" ...
for cfg in "$@"; do
  set -- $cfg
  BH_PULL_SW_CFG_V=$1 BH_PULL_SW_CFG_U=$2 python bench.py --no-cpu --no-fp64 --steps 5 --warmup 3 > gpurun_out/bench_p.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_p.json')); r=d['roofline']
print('V=$1 U=$2', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3])"
done
