# Row-flag pull A/B at c2 (fp32, 64 slots): tools/r02_rf_ab.sh > gpurun_out/rf_ab.txt
one() {  # label, env...
  label=$1; shift
  env "$@" python bench.py --no-cpu --no-fp64 --no-c3 --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench_l.json 2>gpurun_out/bench_l.err || { echo "$label FAILED"; tail -3 gpurun_out/bench_l.err; return; }
  python -c "
import json; d=json.load(open('gpurun_out/bench_l.json')); r=d['roofline']
print('$label', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3], 'frac', round(r['frac'],3))"
}
one sw BH_PULL=sw
for g in 0 1 2; do one rf_g$g BH_RF_GEO=$g,$g; done
