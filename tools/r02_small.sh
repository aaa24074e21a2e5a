set -u
for cl in 4 8 16; do
  echo "CL=$cl"; BH_SMALL_CL=$cl timeout 300 python tools/small_profile.py 2>&1 | tail -2
done
echo "CL=8 no staging"; BH_SMALL_NOSTAGE=1 timeout 300 python tools/small_profile.py 2>&1 | tail -2
BH_SMALL_PROF=1 timeout 300 python tools/small_phases.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_scale.py -q -x 2>&1 | tail -3
