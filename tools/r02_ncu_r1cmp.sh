set -u
M=gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,dram__bytes_read.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active
for t in r1 cur; do
  if [ $t = cur ]; then d=.; else d=_wt_$t; fi
  (cd $d && BH_NO_GRAPH=1 timeout 600 ncu --metrics $M --clock-control none --profile-from-start off -k regex:k_pull_sw --launch-skip 200 --launch-count 4 --csv python tools/prof_step.py --config c2 > /tmp/ncu_$t.csv 2>/dev/null; grep -v "^==" /tmp/ncu_$t.csv | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]
for r in rows[1:]:
    print('$t', r[h.index('Kernel Name')][:45], r[h.index('Metric Name')], r[h.index('Metric Value')])
")
done
