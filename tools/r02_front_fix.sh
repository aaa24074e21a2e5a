set -u
BH_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:"k_front_mark" \
  --launch-skip 0 --launch-count 8 --csv python tools/front_step.py 2>/dev/null | grep -v "^==" | grep "gpu__time" | cut -c1-200
timeout 600 python -m pytest tests/test_gpu_frontier.py -q -x 2>&1 | tail -1
timeout 600 python tools/latency.py --configs c2 c3 --limits 0.01 0.05 -1 2>/dev/null
