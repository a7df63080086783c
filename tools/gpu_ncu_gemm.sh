# source-level ncu capture of the fused step-1 GEMM at the C2 shape + C2 launch list
timeout 600 python tools/pass_probe.py > gpurun_out/pass_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_corr_tc2 -c 1 -o gpurun_out/prof_gemm python tools/pass_probe.py > gpurun_out/ncu_gemm.log 2>&1; echo ncu rc=$?
python tools/profile_step.py c2 2 > gpurun_out/step_plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/launches_c2.csv \
    python tools/profile_step.py c2 2 > gpurun_out/ncu_step_c2.log 2>&1; echo launches rc=$?
