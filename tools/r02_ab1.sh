set -u
mkdir -p gpurun_out
timeout 900 python tools/ab_store.py --config c3 --n 256 > gpurun_out/ab_c3.txt 2>&1; cat gpurun_out/ab_c3.txt
timeout 600 python tools/ab_store.py --config c2 --n 64 --reps 5 --settings BH_RELABEL=1 BH_RELABEL=0 > gpurun_out/ab_c2.txt 2>&1; cat gpurun_out/ab_c2.txt
timeout 600 python -m pytest tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/pytest_scale.txt 2>&1; tail -3 gpurun_out/pytest_scale.txt
