timeout 900 python -m pytest tests/test_gpu_p2p_halo.py -q -p no:cacheprovider -x > gpurun_out/it_p2p.log 2>&1; echo "p2p rc=$?"
tail -30 gpurun_out/it_p2p.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/it_pytest.log
