# quick GPU check: parity suite + one bench line (device, e2e, breakdown)
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
python bench.py --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err || tail -5 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); r=d['roofline']
print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'], 'fp64', d['fp64'] and round(d['fp64']['value'],1))"
