for mb in 8 16 24; do for st in 2 3 4; do
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --max-blocks $mb --streams $st > gpurun_out/r2c_mb${mb}_s${st}.json 2> gpurun_out/r2c_mb${mb}_s${st}.log; echo mb$mb s$st=$? $(python -c "import json;d=json.load(open('gpurun_out/r2c_mb${mb}_s${st}.json'));print(d['ms_per_step'], d['e2e']['ms_per_step'], d['gpu_launches'])")
done; done
