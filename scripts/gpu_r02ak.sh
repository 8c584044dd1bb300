# r02ak: where the tune time goes on the worst config-4 matrices (tridiagonal-like banded)
timeout 600 ncu --nvtx --nvtx-include "so_tune_ml/" --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ak_launches.csv python scripts/tune_cost_probe.py --ids 597,1517 > /dev/null 2>&1; echo rc=$?
