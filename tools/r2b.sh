set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r2b_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_b4.json 2> gpurun_out/r2b_b4.log; echo b4=$?
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2b_ref4.json 2> gpurun_out/r2b_ref4.log; echo ref=$?
