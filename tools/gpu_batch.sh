set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python tools/variants.py --config c2 --n 64 --variants "" "BH_RELABEL=0" > gpurun_out/var_c2.jsonl 2> gpurun_out/var_c2.err; cat gpurun_out/var_c2.jsonl; tail -3 gpurun_out/var_c2.err
timeout 1200 python tools/variants.py --config c3 --n 256 --slots 128 64 --variants "" "BH_L2_PERSIST_MB=0" "BH_RELABEL=0" > gpurun_out/var_c3.jsonl 2> gpurun_out/var_c3.err; cat gpurun_out/var_c3.jsonl; tail -3 gpurun_out/var_c3.err
