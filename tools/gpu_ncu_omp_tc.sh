# source-level ncu capture of the fused tensor-core OMP at the C4 shape
timeout 300 python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/probe.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_omp_tc -s 1 -c 1 -o gpurun_out/omp_tc_src python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/ncu.log 2>&1; echo ncu rc=$?
