# r02l: spread walk with records staged in shared memory for larger matrices (A/B knob SOB_NO_WALK_REC_STAGE)
set -x
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_tuner_corpus.py tests/test_gpu_full_size.py -p no:cacheprovider -k "tune or feature or corpus or predict or spread or config5_stencil512_features" > gpurun_out/l_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/l_pytest.log
IDS=102,150,302,362,30,426,474,90,32,480,360
for i in 1 2; do
SOB_NO_WALK_REC_STAGE=1 timeout 600 python scripts/tune_cost_probe.py --ids $IDS 2>&1 | sed 's/^/global /'
timeout 600 python scripts/tune_cost_probe.py --ids $IDS 2>&1 | sed 's/^/staged /'
done > gpurun_out/l_ab.txt
grep -E 'id": 102|id": 150|wall cost' gpurun_out/l_ab.txt | cut -c1-220
