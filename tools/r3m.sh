# round 3m: config 1 (60-bit specials, mixed integer/FP64 ring) per-op numbers and a per-class profile of tensor+relin
timeout 300 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/r3m_c1.json 2> gpurun_out/r3m_c1.log; echo c1=$?
timeout 300 python tools/kbench.py --config 1 --ops relinb,prof --levels 7 --reps 20 > gpurun_out/r3m_kb.log 2>&1; echo kb=$?
