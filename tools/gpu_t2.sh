timeout 1200 python -m pytest tests/test_gpu_mod_train.py tests/test_gpu_parity_configs.py tests/test_gpu_fused.py -q --timeout 900 -x > gpurun_out/t_mod.log 2>&1; echo tests rc=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; echo bench rc=$?
