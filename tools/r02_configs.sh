# Round-2 configuration table (one B200): every BASELINE config, sampled oracle parity.
set -u
mkdir -p gpurun_out
timeout 600 python tools/run_configs.py --config c1 --dtype fp64 --parity 4 > gpurun_out/r2cfg_c1.json 2>gpurun_out/r2cfg_c1.err; tail -c 300 gpurun_out/r2cfg_c1.json; echo
timeout 600 python tools/run_configs.py --config c2 --parity 8 > gpurun_out/r2cfg_c2.json 2>gpurun_out/r2cfg_c2.err; tail -c 300 gpurun_out/r2cfg_c2.json; echo
timeout 1500 python tools/run_configs.py --config c5 --parity 4 > gpurun_out/r2cfg_c5.json 2>gpurun_out/r2cfg_c5.err; tail -c 300 gpurun_out/r2cfg_c5.json; echo
timeout 1500 python tools/run_configs.py --config c3 --parity 2 > gpurun_out/r2cfg_c3.json 2>gpurun_out/r2cfg_c3.err; tail -c 300 gpurun_out/r2cfg_c3.json; echo
timeout 900 python tools/run_configs.py --config c3 --parity 0 --slots 64 > gpurun_out/r2cfg_c3_64.json 2>gpurun_out/r2cfg_c3_64.err; tail -c 300 gpurun_out/r2cfg_c3_64.json; echo
timeout 2400 python tools/run_configs.py --config c4 --parity 1 > gpurun_out/r2cfg_c4.json 2>gpurun_out/r2cfg_c4.err; tail -c 300 gpurun_out/r2cfg_c4.json; echo
timeout 900 python tools/run_configs.py --config c4 --parity 0 --slots 64 > gpurun_out/r2cfg_c4_64.json 2>gpurun_out/r2cfg_c4_64.err; tail -c 300 gpurun_out/r2cfg_c4_64.json; echo
