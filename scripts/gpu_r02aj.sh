# r02aj: the full 2000-matrix config-4 batch on the final tree: run-first labels + the device ML tuner per matrix
set -x
mkdir -p gpurun_out/c4
timeout 2400 python scripts/config4.py --count 2000 --reps 20 --model paper_2303_05098_b200/models/b200_forest.txt --out gpurun_out/c4/tuned_2000.csv > gpurun_out/c4/run.log 2>&1; echo "config4 rc=$?"
tail -3 gpurun_out/c4/run.log
python scripts/config4_report.py gpurun_out/c4/tuned_2000.csv > gpurun_out/c4/summary_all.json 2>&1; echo "report rc=$?"
python - <<'PY'
import csv, json
ids = set(json.load(open("profiles/config4_split_r02.json"))["test_ids"])
rows = list(csv.DictReader(open("gpurun_out/c4/tuned_2000.csv")))
held = [r for r in rows if int(r["id"]) in ids]
with open("gpurun_out/c4/tuned_heldout.csv", "w", newline="") as f:
    w = csv.DictWriter(f, fieldnames=list(rows[0].keys())); w.writeheader(); w.writerows(held)
print(len(held))
PY
python scripts/config4_report.py gpurun_out/c4/tuned_heldout.csv > gpurun_out/c4/summary_heldout.json 2>&1
cat gpurun_out/c4/summary_all.json
