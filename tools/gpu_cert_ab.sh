timeout 900 python -m pytest tests/test_gpu_certify.py tests/test_gpu_api_fp32.py tests/test_gpu_parity_configs.py -q --timeout 900 -x > gpurun_out/t_cert.log 2>&1; echo tests rc=$?
echo "== sm off" > gpurun_out/cert_ab.log; SDB_CERT_SM=0 timeout 600 python tools/cert_probe.py 2>&1 | tail -1 >> gpurun_out/cert_ab.log
echo "== sm on" >> gpurun_out/cert_ab.log; timeout 600 python tools/cert_probe.py 2>&1 | tail -1 >> gpurun_out/cert_ab.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; echo bench rc=$?
