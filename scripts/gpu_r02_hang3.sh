# Intermittent pageable stall repro (1 GPU): the laplacian loop alone, then after the pinned tests in one process
timeout 600 python scripts/pageable_stall_repro.py 150 > gpurun_out/hg3_a.log 2> gpurun_out/hg3_a.err; echo "a rc=$?"; tail -3 gpurun_out/hg3_a.log; tail -40 gpurun_out/hg3_a.err | grep -v "^round" ; tail -2 gpurun_out/hg3_a.err
for i in 1 2 3 4 5 6 7 8 9 10; do
  timeout 300 python -X faulthandler -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -o faulthandler_timeout=60 -k "coo or pinned or follow or hdc or host" > gpurun_out/hg3_b_$i.log 2>&1; rc=$?; echo "b $i rc=$rc $(tail -1 gpurun_out/hg3_b_$i.log)"
  [ $rc -ne 0 ] && head -80 gpurun_out/hg3_b_$i.log
done
