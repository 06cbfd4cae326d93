# round 6n: ModUp coefficient tiles per block (TG_MODUP_TILES; 1 = one tile per block as before)
TG_MODUP_TILES=4 timeout 900 python -m pytest tests/test_gpu_ksfused.py tests/test_gpu_parity.py tests/test_gpu_pfe.py -q -x > gpurun_out/r6n_new.log 2>&1; echo new=$?; tail -1 gpurun_out/r6n_new.log
run() { env "$@" timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r6n_tmp.json 2>gpurun_out/r6n_tmp.log; echo "$@" $(python -c "import json;d=json.load(open('gpurun_out/r6n_tmp.json'));r=d['roofline']['per_kernel'];print(d['ms_per_step'], d['e2e']['ms_per_step'], d['check']['decrypted_count'], d['clocks']['sm_mhz'], d['gpu_time']['kernel_sum_ms'], {k:round(v['ms'],2) for k,v in r.items() if v['ms']>1})"); }
for t in 1 2 4 8 1 4; do run TG_MODUP_TILES=$t; done
