# round 4g: every config on the current tree (bench lines for profiles/), config-4 reference arm
timeout 600 python bench.py > gpurun_out/r4g_b4.json 2> gpurun_out/r4g_b4.log; echo b4=$?
for c in 3 5 2 1; do timeout 600 python bench.py --config $c > gpurun_out/r4g_b$c.json 2> gpurun_out/r4g_b$c.log; echo b$c=$?; done
