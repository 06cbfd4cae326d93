# round 2 (session 2) evidence: GPU suite, bench lines of every config, config-4 launch list + DRAM traffic,
# ncu --set full of one batched level-21 relinearisation (current kernels)
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/ev_pytest.log
timeout 600 python bench.py > gpurun_out/ev_b4.json 2> gpurun_out/ev_b4.log; echo b4=$?
for c in 3 5 2 1; do timeout 600 python bench.py --config $c > gpurun_out/ev_b$c.json 2> gpurun_out/ev_b$c.log; echo b$c=$?; done
TG_PROFILE_REGION=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev_launches_c4.csv 2> gpurun_out/ev_launches_c4.log; echo launches=$?
TG_PROFILE_REGION=1 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -o gpurun_out/ev_relin_b8 -f python tools/kbench.py --config 4 --ops relinb --levels 21 --reps 1 > gpurun_out/ev_relin_ncu.log 2>&1; echo full=$?
