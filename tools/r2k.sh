timeout 900 python -m pytest tests/test_gpu_protocol.py tests/test_gpu_bootstrap.py tests/test_gpu_pfe.py -x -q > gpurun_out/r2k_pytest.log 2>&1; echo pytest=$?; tail -30 gpurun_out/r2k_pytest.log
