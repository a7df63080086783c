timeout 300 python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_omp_tc -s 7 -c 1 -o gpurun_out/prof_omp_tc2 \
    python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/ncu_omp_tc.log 2>&1; echo ncu rc=$?
