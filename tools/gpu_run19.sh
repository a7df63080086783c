timeout 900 python -m pytest tests -q -m gpu --timeout 900 --deselect tests/test_gpu_parity_configs.py > gpurun_out/gputest2.log 2>&1; echo all rc=$?
timeout 1800 python -m pytest tests/test_gpu_parity_configs.py -q --timeout 1700 > gpurun_out/t_parity.log 2>&1; echo parity rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cert.json 2> gpurun_out/bench_cert.err; echo bench rc=$?
