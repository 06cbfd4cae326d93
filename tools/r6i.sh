# round 6i: ncu --set full of the session-3 kernels inside one timed config-4 step (40 launches after the first 150)
TG_PROFILE_REGION=1 timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off --launch-skip 150 --launch-count 40 -o gpurun_out/r6i_step_c4 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --streams 1 > gpurun_out/r6i_ncu.log 2>&1; echo full=$?
ls -la gpurun_out/r6i_step_c4.ncu-rep
