timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_certify.py -q --timeout 900 > gpurun_out/t_fused.log 2>&1; echo fused rc=$?
timeout 1800 python -m pytest tests/test_gpu_parity_configs.py -q -k "c2" --timeout 1700 > gpurun_out/t_parity.log 2>&1; echo parity rc=$?
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc=$?
