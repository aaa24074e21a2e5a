# plan balance A/B: cost of a row in edges (BH_ROWCOST), c2 fp32 and fp64
one() {  # label, bench args, env...
  label=$1; shift; args=$1; shift
  env "$@" python bench.py --no-cpu --no-fp64 --no-c3 $args > gpurun_out/bench_l.json 2>gpurun_out/bench_l.err || { echo "$label FAILED"; tail -3 gpurun_out/bench_l.err; return; }
  python -c "
import json; d=json.load(open('gpurun_out/bench_l.json')); r=d['roofline']
print('$label', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3], 'slots', d['config'].get('slots'))"
}
for c in "$@"; do
  one "f32 rowcost $c" "--steps 5 --warmup 3" BH_ROWCOST=$c
done
