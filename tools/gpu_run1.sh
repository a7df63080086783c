set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/gputest.log 2>&1; echo pytest rc=$?
timeout 300 python tools/omp_tc_probe.py > gpurun_out/omp_tc_c4.log 2>&1; echo probe rc=$?
timeout 300 python tools/omp_tc_probe.py 1 1000000 256 8 64 > gpurun_out/omp_tc_c5.log 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4 rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2 rc=$?
