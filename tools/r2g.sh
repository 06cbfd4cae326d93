TG_PROFILE_REGION=1 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -o gpurun_out/r2g_relinb -f python tools/kbench.py --config 4 --ops relinb --levels 21 --reps 1 > gpurun_out/r2g_ncu.log 2>&1; echo ncu=$?
ls -la gpurun_out/
