timeout 1200 python -m pytest tests/test_gpu_upload.py tests/test_gpu_api_fp32.py -q --timeout 900 > gpurun_out/t_up.log 2>&1; echo tests rc=$?
