make -j8 >/dev/null 2>&1 || make -j8
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_c4p.csv python scripts/config4.py --count 12 --reps 2 --only scripts/c4_ids_powerlaw.json --model paper_2303_05098_b200/models/b200_forest.txt --out gpurun_out/c4_p.csv > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_c4p.csv')))
st=next(i for i,r in enumerate(rows) if r and r[0]=='ID'); h=rows[st]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size'); mi=h.index('Metric Name'); ii=h.index('ID')
from collections import OrderedDict
per=OrderedDict()
for r in rows[st+1:]:
    if len(r)!=len(h): continue
    per.setdefault(r[ii],[r[ki].split('(')[0].split('::')[-1][:40], r[gi], {}])[2][r[mi]]=float(r[vi].replace(',',''))
items=list(per.values())
for name,g,m in items[-12:]: print(f"{name:42s} {m.get('gpu__time_duration.sum',0)/1e3:9.1f} us dram {(m.get('dram__bytes_read.sum',0)+m.get('dram__bytes_write.sum',0))/1e6:8.1f} MB grid {g}")
PY
cat gpurun_out/c4_p.csv | cut -d, -f1-4,21-
