timeout 900 python -m pytest tests/test_gpu_omp_tc.py tests/test_gpu_certify.py -q --timeout 900 > gpurun_out/t_tc.log 2>&1; echo tc rc=$?
timeout 600 python tools/cert_probe.py > gpurun_out/cert_probe.log 2>&1; echo probe rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/bench_cert.json 2> gpurun_out/bench_cert.err; echo bench rc=$?
