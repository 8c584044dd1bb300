make -j8 >/dev/null 2>&1 || make -j8
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/config4.py --count 12 --reps 2 --model paper_2303_05098_b200/models/b200_forest.txt --out gpurun_out/c4_small.csv > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
from collections import defaultdict
rows=list(csv.reader(open('gpurun_out/launches_c4.csv')))
st=next(i for i,r in enumerate(rows) if r and r[0]=='ID'); h=rows[st]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size')
seq=[(r[ki].split('(')[0].split('::')[-1][:40], float(r[vi].replace(',','')), r[gi]) for r in rows[st+1:] if len(r)==len(h)]
# print the feature pipeline of the last tune calls
for name,t,g in seq[-60:]: print(f"{name:42s} {t/1e3:9.1f} us grid {g}")
PY
cat gpurun_out/c4_small.csv | cut -d, -f1-4,21- | head -14
