# C2 A/B: the C2 job with each library (SDB_LIB), eager per-phase breakdown; GEMM / fused tests with the last one
for lib in "$@"; do
  echo "== $lib"
  SDB_LIB=$lib timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err || tail -3 gpurun_out/bench_ab.err
  python tools/show_bench.py gpurun_out/bench_ab.json | grep -E "ms/step|step1|omp_deferred|certify|mod_update"
done
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fused.py -x -q > gpurun_out/t_tc.log 2>&1; echo tctests rc=$?; tail -2 gpurun_out/t_tc.log
