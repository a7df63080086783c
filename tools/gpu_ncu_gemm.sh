# source-level ncu capture of the fused step-1 GEMM and the deferred OMP at the C2 shape
timeout 600 python tools/pass_probe.py > gpurun_out/pass_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_corr_tc2 -c 1 -o gpurun_out/prof_gemm python tools/pass_probe.py > gpurun_out/ncu_gemm.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_omp_fast -c 1 -o gpurun_out/prof_defer python tools/pass_probe.py > gpurun_out/ncu_defer.log 2>&1; echo ncu rc=$?
