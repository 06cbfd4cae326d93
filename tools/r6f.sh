# round 6f: coarser NTT grids (TG_NTT_BPS grid blocks per SM aimed at; default 4)
run() { env "$@" timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r6f_tmp.json 2>gpurun_out/r6f_tmp.log; echo "$@" $(python -c "import json;d=json.load(open('gpurun_out/r6f_tmp.json'));r=d['roofline']['per_kernel'];print(d['ms_per_step'], d['e2e']['ms_per_step'], d['check']['decrypted_count'], d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in r.items() if v['ms']>1})"); }
for b in 4 3 2 6 4 3 2; do run TG_NTT_BPS=$b; done
