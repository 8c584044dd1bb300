# r02ae: launch list of one steady-state tune_ml on config 3 (R-MAT) and config 2 (NVTX filter so_tune_ml)
timeout 900 ncu --nvtx --nvtx-include "so_tune_ml/" --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ae_tune_launches.csv python scripts/tune_rmat_probe.py > gpurun_out/ae.log 2>&1; echo "rc=$?"
