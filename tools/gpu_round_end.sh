# what the driver runs at round end: full GPU suite, smoke, both bench arms
s=$(date +%s)
timeout 3000 python -m pytest tests -x -q -m gpu > gpurun_out/gputest_full.log 2>&1; echo gputest rc=$? $(( $(date +%s)-s ))s
s=$(date +%s)
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? $(( $(date +%s)-s ))s
s=$(date +%s)
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$? $(( $(date +%s)-s ))s
s=$(date +%s)
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$? $(( $(date +%s)-s ))s
