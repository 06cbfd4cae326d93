# round 6h: 16-warp fused key-switch blocks, two polys side by side sharing the staged twiddles (TG_KS_W16=1)
TG_KS_W16=1 timeout 600 python -m pytest tests/test_gpu_ksfused.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r6h_new.log 2>&1; echo new=$?; tail -1 gpurun_out/r6h_new.log
for t in 1 0 1 0; do TG_KS_W16=$t timeout 300 python tools/kbench.py --config 4 --ops relinb --levels 20,14,9 --reps 20 > gpurun_out/r6h_kb_$t.json 2> gpurun_out/r6h_kb_$t.log; echo kb w16=$t $(tail -c 600 gpurun_out/r6h_kb_$t.json | tr '\n' ' '); done
run() { env "$@" timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r6h_tmp.json 2>gpurun_out/r6h_tmp.log; echo "$@" $(python -c "import json;d=json.load(open('gpurun_out/r6h_tmp.json'));r=d['roofline']['per_kernel'];print(d['ms_per_step'], d['e2e']['ms_per_step'], d['check']['decrypted_count'], d['clocks']['sm_mhz'], {k:round(v['ms'],2) for k,v in r.items() if v['ms']>1})"); }
run TG_KS_W16=1
run TG_KS_W16=0
run TG_KS_W16=1
run TG_KS_W16=0
