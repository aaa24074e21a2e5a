set -u
timeout 600 python tools/run_configs.py --config c5 --parity 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c5', [(r['eps'], round(r['queries_per_s'],1)) for r in d['runs']])"
for c in "" "BH_PULL_CFG_U=6,3"; do
  echo "== c3 $c"; env $c timeout 900 python tools/run_configs.py --config c3 --parity 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['runs'][0]; print('c3', round(r['queries_per_s'],1), r['rounds'], r['slots'])"
done
timeout 900 python tools/run_configs.py --config c4 --parity 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['runs'][0]; print('c4', round(r['queries_per_s'],1), r['rounds'], r['slots'])"
