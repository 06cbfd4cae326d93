# round 6k: pipelines / batch size sweep on the session-3 kernels (default: --streams 4 --max-blocks 8), gadget re-check
run() { timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/r6k_tmp.json 2>gpurun_out/r6k_tmp.log; echo "$@" $(python -c "import json;d=json.load(open('gpurun_out/r6k_tmp.json'));print(d['ms_per_step'], d['e2e']['ms_per_step'], d['check']['decrypted_count'], d['clocks']['sm_mhz'], d['gpu_time']['single_stream_ms'], d['gpu_time']['kernel_sum_ms'])"); }
run --streams 4 --max-blocks 8
run --streams 3 --max-blocks 8
run --streams 6 --max-blocks 8
run --streams 6 --max-blocks 4
run --streams 8 --max-blocks 4
run --streams 4 --max-blocks 16
run --streams 4 --max-blocks 8
run --streams 4 --max-blocks 8 --group 8 --K 8
run --streams 4 --max-blocks 8 --group 6 --K 6
