timeout 900 python -m pytest tests/test_gpu_mod_train.py tests/test_host_logic.py -q --timeout 900 -x > gpurun_out/t_train.log 2>&1; echo tests rc=$?
for k in 1 2 3; do timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_rep$k.json 2> gpurun_out/bench_rep$k.err; echo bench$k rc=$?; done
