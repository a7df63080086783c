timeout 600 python tools/cert_probe.py > gpurun_out/cert_probe.log 2>&1; echo probe rc=$?
timeout 900 python -m pytest tests/test_gpu_certify.py -q --timeout 600 > gpurun_out/t_cert.log 2>&1; echo cert rc=$?
timeout 900 python -m pytest tests -q -m gpu --timeout 900 --deselect tests/test_gpu_parity_configs.py > gpurun_out/gputest2.log 2>&1; echo all rc=$?
