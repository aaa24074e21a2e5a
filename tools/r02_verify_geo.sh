set -u
for dt in fp32 fp64; do echo "== c2 $dt"; timeout 300 python tools/ab_store.py --config c2 --n 64 --reps 5 --dtype $dt --settings "X=1" 2>&1 | grep "q/s"; done
echo "== c5"; timeout 300 python tools/c5_profile.py --n 8192 --eps 1e-4 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/v_pytest.txt 2>&1; tail -2 gpurun_out/v_pytest.txt
