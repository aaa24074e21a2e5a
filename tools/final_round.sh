set -u
python -m pytest tests -m gpu -q 2>&1 | tail -1 > gpurun_out/final_pytest.txt
bash tools/measure_round.sh > gpurun_out/final_measure.log 2>&1
bash tools/run_all_configs.sh > gpurun_out/final_configs.log 2>&1
echo done
