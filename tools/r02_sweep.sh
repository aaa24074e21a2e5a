set -u
for dt in fp32 fp64; do
for c in "" "BH_PULL_CFG_V=8,4" "BH_PULL_CFG_V=6,4" "BH_PULL_CFG_V=5,4" "BH_PULL_CFG_V=6,3" "BH_PULL_CFG_V=8,3" "BH_PULL_CFG_U=6,4" "BH_PULL_CFG_U=7,4" "BH_PULL_CFG_U=5,4" "BH_PULL_CFG_U=8,3" "BH_PULL_CFG_U=6,3"; do
  echo "== c2 $dt $c"; env $c timeout 300 python tools/ab_store.py --config c2 --n 64 --reps 5 --dtype $dt --settings "X=1" 2>&1 | grep "q/s"
done
done
for c in "" "BH_PULL_CFG_V=10,2" "BH_PULL_CFG_V=6,3" "BH_PULL_CFG_V=10,3" "BH_PULL_CFG_U=10,3" "BH_PULL_CFG_U=10,2"; do
  echo "== c5 $c"; env $c timeout 300 python tools/c5_profile.py --n 8192 --eps 1e-4 2>&1 | tail -2
done
