set -x
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu.txt 2>&1; tail -14 gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python tools/run_configs.py --config c1 --dtype fp64 --parity 1 > gpurun_out/cfg_c1.json 2> gpurun_out/cfg_c1.err; cat gpurun_out/cfg_c1.json; tail -3 gpurun_out/cfg_c1.err
BH_NO_SMALL=1 timeout 300 python tools/run_configs.py --config c1 --dtype fp64 --parity 1 > gpurun_out/cfg_c1_engine.json 2>&1; tail -1 gpurun_out/cfg_c1_engine.json
BH_NO_GRAPH=1 timeout 600 python tools/prof_step.py --config c3 --n 64 --slots 64 > gpurun_out/prof_c3_plain.log 2>&1 && \
BH_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_push|k_pull|k_combine|k_control" -s 8 -c 5 -o gpurun_out/prof_c3 python tools/prof_step.py --config c3 --n 64 --slots 64 > gpurun_out/ncu_c3.log 2>&1; tail -3 gpurun_out/ncu_c3.log
