# round 6g: the A/B switches' fallback paths stay bit-exact (full GPU suite with every session-3 fusion off),
# then the evidence of the final kernels: launch list + DRAM traffic of one config-4 step, bench lines, reference arm
TG_LAZY_FUSED=0 TG_FUSED_LADDER=0 TG_MULTI_BASE=0 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r6g_pytest_off.log 2>&1; echo pytest_off=$?; tail -1 gpurun_out/r6g_pytest_off.log
TG_LAZY_RELIN=0 timeout 900 python -m pytest tests/test_gpu_statement.py tests/test_gpu_fullsize.py tests/test_gpu_bsgs.py -q -x > gpurun_out/r6g_pytest_eager.log 2>&1; echo pytest_eager=$?; tail -1 gpurun_out/r6g_pytest_eager.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r6g_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/r6g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r6g_b4.json 2> gpurun_out/r6g_b4.log; echo b4=$?
TG_PROFILE_REGION=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r6g_launches_c4.csv 2> gpurun_out/r6g_launches_c4.log; echo ncu=$?
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/r6g_b1.json 2> gpurun_out/r6g_b1.log; echo b1=$?
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/r6g_b2.json 2> gpurun_out/r6g_b2.log; echo b2=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r6g_ref4.json 2> gpurun_out/r6g_ref4.log; echo ref=$?
