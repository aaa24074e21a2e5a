set -u
for t in r1 5f29d5f cur; do
  if [ $t = cur ]; then d=.; else d=_wt_$t; fi
  echo "== $t"; (cd $d && timeout 600 python tools/c5_profile.py --n 8192 --eps 1e-4 2>&1 | tail -2)
done
