set -u
mkdir -p gpurun_out
timeout 600 python tools/ab_store.py --config c2 --n 64 --reps 5 --settings BH_ELEM_VAR=0 BH_ELEM_VAR=1 BH_ELEM_VAR=2 > gpurun_out/ab2_c2.txt 2>&1; cat gpurun_out/ab2_c2.txt
timeout 600 python tools/ab_store.py --config c2 --n 64 --reps 5 --dtype fp64 --settings BH_ELEM_VAR=0 BH_ELEM_VAR=1 > gpurun_out/ab2_c2d.txt 2>&1; cat gpurun_out/ab2_c2d.txt
timeout 900 python tools/ab_store.py --config c3 --n 256 --settings BH_ELEM_VAR=0 BH_ELEM_VAR=1 BH_ELEM_VAR=2 BH_ELEM_VAR=3 > gpurun_out/ab2_c3.txt 2>&1; cat gpurun_out/ab2_c3.txt
