# quick correctness + speed check after a kernel change
timeout 900 python -m pytest tests -q -m gpu --timeout 900 --deselect tests/test_gpu_parity_configs.py > gpurun_out/gputest.log 2>&1; echo all rc=$?
timeout 1500 python -m pytest tests/test_gpu_parity_configs.py -q -k "c3 or c4" --timeout 1400 > gpurun_out/t_parity.log 2>&1; echo parity rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; echo bench rc=$?
