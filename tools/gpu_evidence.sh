# evidence set: default bench (driver contract), reference arm, C4 + C2 launch lists, ncu of the two top kernels
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
python tools/profile_step.py c4 2 > gpurun_out/step_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c4.csv \
    python tools/profile_step.py c4 2 > gpurun_out/ncu_step.log 2>&1; echo launches c4 rc=$?
python tools/profile_step.py c2 2 > gpurun_out/step_plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c2.csv \
    python tools/profile_step.py c2 2 > gpurun_out/ncu_step_c2.log 2>&1; echo launches c2 rc=$?
python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_omp_tc -s 7 -c 1 -o gpurun_out/prof_omp_tc \
    python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/ncu_omp_tc.log 2>&1; echo ncu1 rc=$?
python tools/cert_probe.py > gpurun_out/cert_probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_certify -s 2 -c 1 -o gpurun_out/prof_cert \
    python tools/cert_probe.py > gpurun_out/ncu_cert.log 2>&1; echo ncu2 rc=$?
