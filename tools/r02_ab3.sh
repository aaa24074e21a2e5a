set -u
mkdir -p gpurun_out
: > gpurun_out/ab3_c3.txt
for s in "" "BH_L2_PERSIST_MB=0" "BH_L2_PERSIST_MB=0 BH_RELABEL=0"; do
  for slots in 128 64 32; do
    env $s timeout 600 python tools/ab_store.py --config c3 --n 256 --reps 1 --slots $slots --settings "BH_X=$slots" 2>&1 | grep "q/s" | sed "s/^/[$s] /" >> gpurun_out/ab3_c3.txt
  done
done
cat gpurun_out/ab3_c3.txt
