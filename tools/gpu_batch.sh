set -x
free -g | head -2; nproc
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_baselines.py -x -q --durations=20 > gpurun_out/pytest_cfg.txt 2>&1; tail -30 gpurun_out/pytest_cfg.txt
timeout 1200 python tools/variants.py --config c3 --n 256 --slots 64 --variants "" "BH_ELEM_VAR=0" "BH_ELEM_VAR=2" "BH_ELEM_VAR=3" > gpurun_out/var_c3e.jsonl 2> gpurun_out/var_c3e.err; cat gpurun_out/var_c3e.jsonl; tail -3 gpurun_out/var_c3e.err
timeout 600 python tools/variants.py --config c3 --n 256 --slots 32 128 > gpurun_out/var_c3b.jsonl 2> gpurun_out/var_c3b.err; cat gpurun_out/var_c3b.jsonl; tail -3 gpurun_out/var_c3b.err
