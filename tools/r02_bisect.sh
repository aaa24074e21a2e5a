set -u
for t in r1 5f29d5f 3f001b3 a7be422 584521f cur; do
  if [ $t = cur ]; then d=.; else d=_wt_$t; fi
  (cd $d && timeout 600 python tools/run_configs.py --config c5 --eps 1e-4 --parity 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['runs'][0]; print('$t c5 1e-4', round(r['queries_per_s'],1), r['rounds'])")
done
