timeout 2400 python tools/sweep_c5.py > gpurun_out/c5_sweep.json 2> gpurun_out/c5_sweep.err; echo sweep rc=$?
timeout 600 python tools/profile_step.py c2 1 > gpurun_out/step_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_corr_tc2 -s 4 -c 1 -o gpurun_out/prof_corr python tools/profile_step.py c2 1 > gpurun_out/ncu_corr.log 2>&1; echo ncu rc=$?
