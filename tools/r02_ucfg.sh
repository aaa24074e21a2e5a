set -u
echo "== r1"; (cd _wt_r1 && timeout 300 python tools/c5_profile.py --n 8192 --eps 1e-4 2>&1 | tail -2)
for c in "" "BH_PULL_CFG_U=8,2" "BH_PULL_CFG_U=5,3" "BH_PULL_CFG_U=8,3" "BH_PULL_CFG_U=4,4" "BH_PULL_CFG_U=6,4" "BH_PULL_CFG_V=6,3" "BH_PULL_CFG_V=8,3"; do
  echo "== cur $c"; env $c timeout 300 python tools/c5_profile.py --n 8192 --eps 1e-4 2>&1 | tail -2
done
