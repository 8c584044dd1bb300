timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/it_pytest.log
LAB_ONLY_PROD=1 LAB_PEAK=6539.5 timeout 600 ./build/lab band,lap,rmat > gpurun_out/it_lab.log 2>&1; echo "lab rc=$?"
cat gpurun_out/it_lab.log
LAB_ONLY_PROD=1 LAB_REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it_lab_ncu.csv ./build/lab rmat > /dev/null 2>&1; echo "ncu rc=$?"
python3 - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/it_lab_ncu.csv')))
st=next(i for i,r in enumerate(rows) if r and r[0]=='ID'); h=rows[st]
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
from collections import defaultdict
agg=defaultdict(list)
for r in rows[st+1:]:
    if len(r)==len(h): agg[r[ki].split('(')[0][-60:]].append(float(r[vi].replace(',','')))
for k,v in agg.items(): print(f"{k:60s} n={len(v):4d} median {sorted(v)[len(v)//2]/1e3:9.1f} us")
PY
