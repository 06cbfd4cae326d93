# round 6j: tensor operands read in place through poly strides (TG_OPERAND_STRIDES=0: level-dropped views gathered first)
timeout 900 python -m pytest tests/test_gpu_ksfused.py tests/test_gpu_bsgs.py tests/test_gpu_statement.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r6j_new.log 2>&1; echo new=$?; tail -1 gpurun_out/r6j_new.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r6j_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/r6j_pytest.log
run() { env "$@" timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r6j_tmp.json 2>gpurun_out/r6j_tmp.log; echo "$@" $(python -c "import json;d=json.load(open('gpurun_out/r6j_tmp.json'));r=d['roofline']['per_kernel'];print(d['ms_per_step'], d['e2e']['ms_per_step'], d['check']['decrypted_count'], d['clocks']['sm_mhz'], d['gpu_time']['single_stream_ms'], d['gpu_time']['kernel_sum_ms'], {k:round(v['ms'],2) for k,v in r.items() if v['ms']>1})"); }
run TG_OPERAND_STRIDES=1
run TG_OPERAND_STRIDES=0
run TG_OPERAND_STRIDES=1
run TG_OPERAND_STRIDES=0
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r6j_b4_full.json 2> gpurun_out/r6j_b4_full.log; echo full=$?; python -c "import json;d=json.load(open('gpurun_out/r6j_b4_full.json'));print(d['ms_per_step'], d['cpu_baseline']['bit_exact_vs_oracle_bsgs'])"
# ncu --set full of 24 launches inside one timed single-stream step, summarised on the box (the report stays there)
TG_PROFILE_REGION=1 timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off --launch-skip 150 --launch-count 24 -o /tmp/r6j_step_c4 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --streams 1 > gpurun_out/r6j_ncu.log 2>&1; echo ncu=$?
python tools/ncu_summary.py /tmp/r6j_step_c4.ncu-rep > gpurun_out/r6j_ncu_summary.md 2> gpurun_out/r6j_ncu_summary.err; echo summary=$?
for k in k_mod_down_fp kw_ks_chunks; do ncu -i /tmp/r6j_step_c4.ncu-rep --page source --csv --kernel-name regex:$k --launch-count 1 --print-source sass > /tmp/r6j_$k.csv 2>/dev/null; echo "## $k" >> gpurun_out/r6j_stalls.md; python tools/ncu_sass_stalls.py /tmp/r6j_$k.csv >> gpurun_out/r6j_stalls.md 2>> gpurun_out/r6j_stalls.err; done; echo stalls=$?
