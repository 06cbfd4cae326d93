# round 6r: ciphertext stacking / part gathers as one launch (was one device copy per poly)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r6r_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/r6r_pytest.log
run() { env "$@" timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r6r_tmp.json 2>gpurun_out/r6r_tmp.log; echo "$@" $(python -c "import json;d=json.load(open('gpurun_out/r6r_tmp.json'));print(d['ms_per_step'], d['e2e']['ms_per_step'], d['check']['decrypted_count'], d['clocks']['sm_mhz'], d['gpu_time']['single_stream_ms'], d['gpu_time']['kernel_sum_ms'], d['gpu_launches'])"); }
run TG_X=1
run TG_X=1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r6r_b4.json 2> gpurun_out/r6r_b4.log; echo full=$?; python -c "import json;d=json.load(open('gpurun_out/r6r_b4.json'));print(d['ms_per_step'], d['e2e']['ms_per_step'], d['cpu_baseline']['bit_exact_vs_oracle_bsgs'], d['clocks'])"
timeout 400 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/r6r_b3.json 2> gpurun_out/r6r_b3.log; python -c "import json;d=json.load(open('gpurun_out/r6r_b3.json'));print('c3', d['ms_per_step'], d['e2e']['ms_per_step'], d['cpu_baseline']['bit_exact_vs_oracle_bsgs'])"
