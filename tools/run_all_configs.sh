# All BASELINE configurations through tools/run_configs.py (one B200); JSON per config in gpurun_out/.
set -u
timeout 900 python tools/run_configs.py --config c1 --dtype fp64 --parity 1 > gpurun_out/cfg_c1.json 2>gpurun_out/cfg_c1.err
timeout 1500 python tools/run_configs.py --config c5 --parity 4 > gpurun_out/cfg_c5.json 2>gpurun_out/cfg_c5.err
timeout 1500 python tools/run_configs.py --config c3 --parity 3 --lambda-check > gpurun_out/cfg_c3.json 2>gpurun_out/cfg_c3.err
timeout 2400 python tools/run_configs.py --config c4 --parity 1 > gpurun_out/cfg_c4.json 2>gpurun_out/cfg_c4.err
echo done
