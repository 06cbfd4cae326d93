timeout 600 python -m pytest tests/test_gpu_bsgs.py -q -x > gpurun_out/r6q.log 2>&1; echo bsgs=$?; tail -2 gpurun_out/r6q.log
