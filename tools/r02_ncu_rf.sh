# ncu --set full of one mid-batch round's row-flag pulls at c2 (fp32, 64 slots), source-level.
set -u
mkdir -p gpurun_out
BH_NO_GRAPH=1 timeout 300 python tools/prof_step.py --config c2 > gpurun_out/prof_c2_plain.log 2>&1 || { tail -5 gpurun_out/prof_c2_plain.log; exit 1; }
BH_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"k_pull_rf|k_pull_sw" --launch-skip ${SKIP:-120} --launch-count 2 -o gpurun_out/${NAME:-ncu_c2_rf} -f \
  python tools/prof_step.py --config c2 > gpurun_out/ncu_c2_rf.log 2>&1; tail -3 gpurun_out/ncu_c2_rf.log
