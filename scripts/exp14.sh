ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/prof_step.py c4 unfused 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/c4_launches.csv')) if len(r)>10]
h=rows[0]; i=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); idi=h.index('ID')
d={}
for r in rows[1:]:
    d.setdefault((r[idi], r[i][:60]), {})[r[mi]]=r[vi]
for (k,n),m in d.items(): print(k, n, m)
PY
