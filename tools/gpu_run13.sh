timeout 900 python -m pytest tests -q -m gpu --timeout 900 --deselect tests/test_gpu_parity_configs.py > gpurun_out/gputest2.log 2>&1; echo all rc=$?
timeout 600 python tools/cert_probe.py > gpurun_out/cert_probe.log 2>&1; echo probe rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cert.json 2> gpurun_out/bench_cert.err; echo bench rc=$?
timeout 2400 python -m pytest tests/test_gpu_parity_configs.py -q --timeout 2000 -k "c4 or c5" > gpurun_out/t_parity.log 2>&1; echo parity rc=$?
