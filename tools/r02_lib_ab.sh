# A/B of library builds: c2 fp32 / fp64 (64 slots) and the 128-slot proxy (c2 graph, 1024 sources)
one() {  # label, bench args, env...
  label=$1; shift; args=$1; shift
  env "$@" python bench.py --no-cpu --no-fp64 --no-c3 $args > gpurun_out/bench_l.json 2>gpurun_out/bench_l.err || { echo "$label FAILED"; tail -3 gpurun_out/bench_l.err; return; }
  python -c "
import json; d=json.load(open('gpurun_out/bench_l.json')); r=d['roofline']
print('$label', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3], 'slots', d['config'].get('slots'))"
}
for lib in "$@"; do
  one "f32/64 $lib" "--steps 5 --warmup 3" BH_LIBBHPP=$lib
  one "f64/64 $lib" "--steps 3 --warmup 3 --dtype fp64" BH_LIBBHPP=$lib
  one "f32/128 $lib" "--steps 3 --warmup 2 --scaling strong --batch 1024 --slots 128" BH_LIBBHPP=$lib
done
