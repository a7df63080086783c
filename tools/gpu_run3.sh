timeout 900 python tools/parity_trace.py c4 10 c4 3 > gpurun_out/trace_c4.jsonl 2> gpurun_out/trace_c4.err
timeout 900 python tools/parity_trace.py c3 17 c2 9 > gpurun_out/trace_c23.jsonl 2> gpurun_out/trace_c23.err
timeout 300 python -m pytest tests/test_gpu_mod_train.py -q -k min_norm > gpurun_out/t_mn.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_new.json 2> gpurun_out/bench_new.err
