# per-side row-flag pull geometry A/B ("v,u"): c2 fp64 (64 slots) and the 128-slot fp32 proxy
one() {  # label, bench args, env...
  label=$1; shift; args=$1; shift
  env "$@" python bench.py --no-cpu --no-fp64 --no-c3 $args > gpurun_out/bench_l.json 2>gpurun_out/bench_l.err || { echo "$label FAILED"; tail -3 gpurun_out/bench_l.err; return; }
  python -c "
import json; d=json.load(open('gpurun_out/bench_l.json')); r=d['roofline']
print('$label', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3], 'slots', d['config'].get('slots'))"
}
for g in "$@"; do
  one "f64/64 geo $g" "--steps 3 --warmup 3 --dtype fp64" BH_RF_GEO=$g
  one "f32/128 geo $g" "--steps 3 --warmup 2 --scaling strong --batch 1024 --slots 128" BH_RF_GEO=$g
done
