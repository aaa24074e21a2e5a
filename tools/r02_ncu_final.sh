# Round-2 ncu evidence (one B200): smoke launch list, bench launch list, full captures of
# the c2 round kernels, the small-path cluster kernel and the frontier kernels.
set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_smoke.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_ncu_smoke.log 2>&1; tail -1 gpurun_out/r2_ncu_smoke.log
BH_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-fp64 --no-c3 > gpurun_out/r2_ncu_bench.log 2>&1; tail -1 gpurun_out/r2_ncu_bench.log
BH_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"k_push|k_pull_rf|k_combine|k_control" --launch-skip 240 --launch-count 5 -o gpurun_out/r2_ncu_c2_round -f \
  python tools/prof_step.py --config c2 > gpurun_out/r2_ncu_c2.log 2>&1; tail -1 gpurun_out/r2_ncu_c2.log
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_small_query" \
  --launch-count 1 -o gpurun_out/r2_ncu_small -f python tools/small_phases.py > gpurun_out/r2_ncu_small.log 2>&1; tail -1 gpurun_out/r2_ncu_small.log
BH_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:"k_front|k_push" \
  --launch-skip 6 --launch-count 6 -o gpurun_out/r2_ncu_front -f python tools/front_step.py > gpurun_out/r2_ncu_front.log 2>&1; tail -1 gpurun_out/r2_ncu_front.log
ls -la gpurun_out/r2_*
