timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r2d_pytest.log
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/r2d_b1.json 2> gpurun_out/r2d_b1.log; echo b1=$?
timeout 600 python bench.py --config 1 --impl reference --steps 2 --warmup 1 > gpurun_out/r2d_ref1.json 2> gpurun_out/r2d_ref1.log; echo ref1=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2d_b4.json 2> gpurun_out/r2d_b4.log; echo b4=$?
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/r2d_b3.json 2> gpurun_out/r2d_b3.log; echo b3=$?
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/r2d_b2.json 2> gpurun_out/r2d_b2.log; echo b2=$?
