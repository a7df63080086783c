set -x
timeout 600 python -m pytest tests/test_gpu_synth.py tests/test_gpu_mod_train.py tests/test_gpu_fused.py -q --timeout 600 > gpurun_out/t_quick.log 2>&1; echo quick rc=$?
timeout 2400 python -m pytest tests/test_gpu_parity_configs.py -q --timeout 2000 -k "c5" > gpurun_out/t_c5.log 2>&1; echo c5 rc=$?
timeout 2400 python -m pytest tests/test_gpu_parity_configs.py -q --timeout 2000 -k "c4" > gpurun_out/t_c4.log 2>&1; echo c4 rc=$?
timeout 2400 python -m pytest tests/test_gpu_parity_configs.py -q --timeout 2000 -k "c2 or c3" --durations=5 > gpurun_out/t_c23.log 2>&1; echo c23 rc=$?
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 --deselect tests/test_gpu_parity_configs.py --durations=15 > gpurun_out/gputest.log 2>&1; echo all rc=$?
