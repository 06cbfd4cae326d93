# round 6e: block scheduling experiments -- special rows first in kw_ks_chunks (TG_KS_REV), grid granularity of the
# NTT kernels (TG_NTT_BPS blocks per SM aimed at) and of the fused core (TG_KS_Z batch split)
run() { env "$@" timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r6e_tmp.json 2>gpurun_out/r6e_tmp.log; echo "$@" $(python -c "import json;d=json.load(open('gpurun_out/r6e_tmp.json'));r=d['roofline']['per_kernel'];print(d['ms_per_step'], d['e2e']['ms_per_step'], d['check']['decrypted_count'], d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in r.items() if v['ms']>1})"); }
timeout 600 python -m pytest tests/test_gpu_ksfused.py -q -x > gpurun_out/r6e_new.log 2>&1; echo new=$?; tail -1 gpurun_out/r6e_new.log
run TG_KS_REV=1
run TG_KS_REV=0
run TG_KS_REV=1
run TG_KS_REV=0
for b in 8 16 32 64; do run TG_NTT_BPS=$b; done
for z in 2 4 8; do run TG_KS_Z=$z; done
run TG_NTT_BPS=16 TG_KS_Z=4
