# c5-style (128 slots) throughput per elementwise geometry: tools/c5_elem.sh "PUSH COMB" ...
for cfg in "$@"; do
  set -- $cfg
  echo "push=$1 comb=$2 $(BH_ELEM_PUSH=$1 BH_ELEM_COMBINE=$2 python tools/c5_profile.py --n 4096 --eps 1e-6 2>/dev/null | tr '\n' ' ')"
done
