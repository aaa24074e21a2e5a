# Round-end measurement set (one B200): bench line, reference arm, launch list, ncu full of one round.
set -u
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -c 300 gpurun_out/bench_final.json; echo
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 300 gpurun_out/bench_ref.json; echo
BH_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-fp64 \
  > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
BH_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  --launch-skip 421 --launch-count 6 -o gpurun_out/prof_round_final python tools/prof_step.py \
  > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
