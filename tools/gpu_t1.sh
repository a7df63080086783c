timeout 1200 python -m pytest tests/test_gpu_certify.py tests/test_gpu_fused.py -q --timeout 900 > gpurun_out/t_cert.log 2>&1; echo tests rc=$?
