# r02m: entry-parallel vs lockstep feature sweep on the config-4 worst cases (A/B knob SOB_FEAT_ENTRY)
IDS=102,150,302,362,30,426,474,90,32,480,360,370,12,444,84
for i in 1 2; do
for e in 0 1; do SOB_FEAT_ENTRY=$e timeout 600 python scripts/tune_cost_probe.py --ids $IDS 2>&1 | sed "s/^/entry$e /"; done
timeout 600 python scripts/tune_cost_probe.py --ids $IDS 2>&1 | sed "s/^/auto /"
done > gpurun_out/m_ab.txt
cat gpurun_out/m_ab.txt | cut -c1-200
