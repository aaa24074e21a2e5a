set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_frontier.py -x -q > gpurun_out/pytest_front.txt 2>&1; tail -3 gpurun_out/pytest_front.txt
for dt in fp32 fp64; do
timeout 600 python tools/ab_store.py --config c2 --n 64 --reps 5 --dtype $dt --settings "BH_PULL=sw" "BH_PULL=lean" "BH_PULL=lean BH_PULL_LEAN=8,3" "BH_PULL=lean BH_PULL_LEAN=12,3" "BH_PULL=lean BH_PULL_LEAN=6,4" > gpurun_out/ab4_c2_$dt.txt 2>&1; cat gpurun_out/ab4_c2_$dt.txt
done
timeout 900 python tools/ab_store.py --config c3 --n 256 --reps 1 --settings "BH_PULL=sw" "BH_PULL=lean" "BH_PULL=lean BH_PULL_LEAN=8,3" > gpurun_out/ab4_c3.txt 2>&1; cat gpurun_out/ab4_c3.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.txt 2>&1; tail -4 gpurun_out/pytest_gpu3.txt
