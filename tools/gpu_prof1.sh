# k_omp_tc capture at the C4 shape + launch list of one C4 training job
python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_omp_tc -s 7 -c 1 -o gpurun_out/prof_omp_tc \
    python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/ncu_omp_tc.log 2>&1
python tools/profile_step.py c4 2 > gpurun_out/step_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c4.csv \
    python tools/profile_step.py c4 2 > gpurun_out/ncu_step.log 2>&1
