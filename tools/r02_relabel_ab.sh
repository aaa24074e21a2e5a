set -u
for r in 1 0 1 0; do
  echo "RELABEL=$r"
  BH_RELABEL=$r timeout 600 python tools/run_configs.py --config c5 --eps 1e-4 --parity 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['runs'][0]; print('c5 1e-4', round(r['queries_per_s'],1), r['rounds'])"
  BH_RELABEL=$r timeout 600 python tools/run_configs.py --config c2 --parity 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['runs'][0]; print('c2', round(r['queries_per_s'],1), r['rounds'])"
done
