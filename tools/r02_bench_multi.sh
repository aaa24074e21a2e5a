# bench.py's multi-rank path on a one-GPU box: 2 ranks pinned to device 0, gloo exchange
set -u
BH_BENCH_DEVICE=0 BH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu --no-c3 --no-fp64 > gpurun_out/bm_weak.json 2> gpurun_out/bm_weak.err; echo "rc=$?"; tail -c 600 gpurun_out/bm_weak.json; tail -3 gpurun_out/bm_weak.err
BH_BENCH_DEVICE=0 BH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --scaling strong --steps 2 --warmup 1 --no-cpu --no-c3 --no-fp64 > gpurun_out/bm_strong.json 2> gpurun_out/bm_strong.err; echo "rc=$?"; tail -c 600 gpurun_out/bm_strong.json; tail -3 gpurun_out/bm_strong.err
timeout 600 python bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bm_ref.json 2> gpurun_out/bm_ref.err; echo "rc=$?"; tail -c 300 gpurun_out/bm_ref.json
