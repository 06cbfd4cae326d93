set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
nproc; lscpu | grep -i "model name"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r2a_pytest.log
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_b4.json 2> gpurun_out/r2a_b4.log; echo b4=$?
for gk in "8 8" "11 11" "6 6"; do set -- $gk; timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --group $1 --K $2 > gpurun_out/r2a_g$1_$2.json 2> gpurun_out/r2a_g$1_$2.log; echo g$1=$?; done
