timeout 600 python scripts/profile_features.py --ids 877 1843 555 165 706 1692 --reps 5 2>&1 | tail -8
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/feat_launches.csv python scripts/profile_features.py --ids 877 1843 165 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
python3 - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/feat_launches.csv')))
st=next(i for i,r in enumerate(rows) if r and r[0]=='ID'); h=rows[st]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size')
for r in rows[st+1:]:
    if len(r)==len(h): print(f"{r[ki].split('(')[0][-45:]:45s} {float(r[vi].replace(',',''))/1e3:9.1f} us  grid {r[gi]}")
PY
