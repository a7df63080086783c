timeout 900 python -m pytest tests/test_gpu_certify.py -q -x --timeout 600 > gpurun_out/t_cert.log 2>&1; echo cert rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity_configs.py -q --timeout 1100 -k "c4" > gpurun_out/t_c4b.log 2>&1; echo c4 rc=$?
timeout 900 python tools/parity_trace.py c4 10 > gpurun_out/trace3.jsonl 2> gpurun_out/trace3.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/bench_cert.json 2> gpurun_out/bench_cert.err; echo bench rc=$?
timeout 900 python -m pytest tests -q -m gpu -x --timeout 900 --deselect tests/test_gpu_parity_configs.py > gpurun_out/gputest2.log 2>&1; echo all rc=$?
