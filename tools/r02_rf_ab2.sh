# Row-flag pull geometry A/B: c2 fp32 (64 slots), c2 fp64, c5 (128 fp32 slots)
one() {  # label, bench args, env...
  label=$1; shift; args=$1; shift
  env "$@" python bench.py --no-cpu --no-fp64 --no-c3 $args > gpurun_out/bench_l.json 2>gpurun_out/bench_l.err || { echo "$label FAILED"; tail -3 gpurun_out/bench_l.err; return; }
  python -c "
import json; d=json.load(open('gpurun_out/bench_l.json')); r=d['roofline']
print('$label', round(d['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'][:3], 'slots', d['config'].get('slots'))"
}
for g in 3 0; do one c2_f32_g$g "--steps 5 --warmup 3" BH_RF_GEO=$g; done
one c2_f64_sw "--steps 3 --warmup 3 --dtype fp64" BH_PULL=sw
for g in 0 1 2 3; do one c2_f64_g$g "--steps 3 --warmup 3 --dtype fp64" BH_RF_GEO=$g; done
one c5_sw "--config c5 --steps 1 --warmup 1" BH_PULL=sw
for g in 0 1 2 3; do one c5_g$g "--config c5 --steps 1 --warmup 1" BH_RF_GEO=$g; done
