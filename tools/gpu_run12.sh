timeout 900 python tools/standard_vs_split.py c4 > gpurun_out/std_c4.json 2> gpurun_out/std_c4.err; echo c4 rc=$?
timeout 900 python tools/standard_vs_split.py c2 > gpurun_out/std_c2.json 2> gpurun_out/std_c2.err; echo c2 rc=$?
timeout 900 python -m pytest tests/test_gpu_cli.py tests/test_gpu_api_fp32.py -q > gpurun_out/t_cli.log 2>&1; echo cli rc=$?
timeout 600 python tools/profile_step.py c4 1 > gpurun_out/step_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_normal_eq -s 8 -c 1 -o gpurun_out/prof_neq python tools/profile_step.py c4 1 > gpurun_out/ncu_neq.log 2>&1; echo ncu rc=$?
