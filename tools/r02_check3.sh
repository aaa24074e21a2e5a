set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_frontier.py tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_front.txt 2>&1; tail -15 gpurun_out/pytest_front.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.txt 2>&1; tail -6 gpurun_out/pytest_gpu4.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.txt 2>&1; tail -2 gpurun_out/smoke4.txt
timeout 900 python bench.py --no-cpu > gpurun_out/bench4.json 2> gpurun_out/bench4.err; python -c "
import json; d=json.load(open('gpurun_out/bench4.json')); r=d['roofline']
print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), {k: round(v,3) for k,v in r['breakdown_ms_per_step'].items()}, r['timed_step_ms'], 'fp64', d['fp64'] and round(d['fp64']['value'],1), 'c3', d.get('hbm_regime',{}).get('value'))" || tail -5 gpurun_out/bench4.err
