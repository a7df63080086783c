timeout 300 python -m pytest tests/test_gpu_omp_tc.py -q -x --timeout 240 > gpurun_out/t_tc.log 2>&1; echo tc rc=$?
timeout 300 python tools/cert_probe.py > gpurun_out/cert_probe.log 2>&1; echo probe rc=$?
