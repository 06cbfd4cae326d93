# round 6m: final session-3 evidence on the committed kernels: GPU suite, smoke, bench lines of every config, reference arm, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r6m_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r6m_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r6m_b4.json 2> gpurun_out/r6m_b4.log; echo b4=$?
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/r6m_b3.json 2> gpurun_out/r6m_b3.log; echo b3=$?
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/r6m_b5.json 2> gpurun_out/r6m_b5.log; echo b5=$?
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/r6m_b2.json 2> gpurun_out/r6m_b2.log; echo b2=$?
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/r6m_b1.json 2> gpurun_out/r6m_b1.log; echo b1=$?
TG_PROFILE_REGION=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r6m_launches_c4.csv 2> gpurun_out/r6m_launches_c4.log; echo ncu=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r6m_ref4.json 2> gpurun_out/r6m_ref4.log; echo ref=$?
