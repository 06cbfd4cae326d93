# round 3d: TC base conversion v6 (warp-specialised): parity + microbench + ncu of the batch-8 launches
timeout 400 python -m pytest tests/test_gpu_parity.py -k tensor_core -q --tb=line 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_ksfused.py tests/test_gpu_statement.py -x -q > gpurun_out/r3e_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/r3e_pytest.log
for t in 1 0; do TG_TC_BASECONV=$t timeout 300 python tools/kbench.py --config 4 --ops relinb --levels 21,14 --reps 20 > gpurun_out/r3e_kb$t.log 2>&1; echo tc=$t; grep -E "modup|mod_down|mul_relin_rescale" gpurun_out/r3e_kb$t.log; done
TG_PROFILE_REGION=1 timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_mod_down_tc|k_modup_tc" --launch-skip 4 -c 2 -o gpurun_out/r3e_tc -f python tools/kbench.py --config 4 --ops relinb --levels 21 --reps 2 > gpurun_out/r3e_ncu.log 2>&1; echo ncu=$?
