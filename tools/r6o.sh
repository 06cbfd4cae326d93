# round 6o: ModUp output-row split (TG_MODUP_GROUPS; default: 1 group for batched launches)
run() { env "$@" timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r6o_tmp.json 2>gpurun_out/r6o_tmp.log; echo "$@" $(python -c "import json;d=json.load(open('gpurun_out/r6o_tmp.json'));r=d['roofline']['per_kernel'];print(d['ms_per_step'], d['e2e']['ms_per_step'], d['check']['decrypted_count'], d['clocks']['sm_mhz'], d['gpu_time']['kernel_sum_ms'], {k:round(v['ms'],2) for k,v in r.items() if v['ms']>1})"); }
for t in 1 2 3 4 1 2; do run TG_MODUP_GROUPS=$t; done
