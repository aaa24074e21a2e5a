set -u
for t in cur r1 cur r1; do
  if [ $t = r1 ]; then d=_wt_r1; else d=.; fi
  (cd $d && timeout 600 python tools/run_configs.py --config c5 --eps 1e-4 --parity 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['runs'][0]; print('$t c5 1e-4', round(r['queries_per_s'],1), r['rounds'])")
  (cd $d && timeout 600 python tools/run_configs.py --config c2 --parity 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['runs'][0]; print('$t c2', round(r['queries_per_s'],1), r['rounds'])")
done
