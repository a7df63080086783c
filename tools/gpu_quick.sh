# after a kernel change: the whole GPU suite, then the C4 and C2 job times (device-resident legs only)
s=$(date +%s)
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputest_full.log 2>&1; echo gputest rc=$? $(( $(date +%s)-s ))s
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; echo bench rc=$?
