# round 6l: config 5 (K = 10 specials): fused FP64 ModDown (rescale / ladder) vs tensor-core ModDown + separate passes
run() { env "$@" timeout 600 python bench.py --config 5 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r6l_tmp.json 2>gpurun_out/r6l_tmp.log; echo "$@" $(python -c "import json;d=json.load(open('gpurun_out/r6l_tmp.json'));r=d['roofline']['per_kernel'];print(d['ms_per_step'], d['check']['decrypted_count'], d['clocks']['sm_mhz'], {k:round(v['ms'],1) for k,v in r.items() if v['ms']>5})"); }
run TG_X=0
run TG_FUSED_LADDER=0
run TG_FUSED_LADDER=0 TG_FUSED_RESCALE=0
run TG_X=0
