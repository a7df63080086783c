# re-entry check: GPU tests, bench, k_omp_tc source-level capture
timeout 900 python -m pytest tests -q -m gpu --timeout 900 --deselect tests/test_gpu_parity_configs.py > gpurun_out/gputest.log 2>&1; echo all rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; echo bench rc=$?
timeout 300 python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/probe.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_omp_tc -c 1 -o gpurun_out/omp_tc_src python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc > gpurun_out/ncu.log 2>&1; echo ncu rc=$?
