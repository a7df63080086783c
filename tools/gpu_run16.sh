timeout 300 python -m pytest tests/test_gpu_omp_tc.py -q -x --timeout 240 > gpurun_out/t_tc.log 2>&1; echo tc rc=$?
timeout 300 python tools/cert_probe.py > gpurun_out/cert_probe.log 2>&1; echo probe rc=$?
SDB_OMP_TC_2GRP=1 timeout 300 python tools/cert_probe.py > gpurun_out/cert_probe_2g.log 2>&1; echo probe2 rc=$?
timeout 600 python -m pytest tests/test_gpu_certify.py tests/test_gpu_parity_configs.py -k "certif or c4" -q --timeout 500 > gpurun_out/t_c4.log 2>&1; echo c4 rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/bench_cert.json 2> gpurun_out/bench_cert.err; echo bench rc=$?
