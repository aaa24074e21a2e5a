# c5-style (128 slots, refilled) throughput per pull geometry: tools/c5_cfg.sh "V U" ...
for cfg in "$@"; do
  set -- $cfg
  echo "V=$1 U=$2 $(BH_PULL_SW_CFG_V=$1 BH_PULL_SW_CFG_U=$2 python tools/c5_profile.py --n 4096 --eps 1e-6 2>/dev/null | head -1)"
done
