# round 3c: pipelined TC base conversion v4: parity + microbench + ncu of batch-8 launches
timeout 400 python -m pytest tests/test_gpu_parity.py -k tensor_core -q --tb=line 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_ksfused.py tests/test_gpu_statement.py -x -q > gpurun_out/r3c_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r3c_pytest.log
TG_TC_BASECONV=1 timeout 300 python tools/kbench.py --config 4 --ops relinb --levels 21,14 --reps 20 > gpurun_out/r3c_kb1.log 2>&1; grep -E "batch8" gpurun_out/r3c_kb1.log
TG_PROFILE_REGION=1 timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_mod_down_tc|k_modup_tc" --launch-skip 4 -c 2 -o gpurun_out/r3c_tc -f python tools/kbench.py --config 4 --ops relinb --levels 21 --reps 2 > gpurun_out/r3c_ncu.log 2>&1; echo ncu=$?
