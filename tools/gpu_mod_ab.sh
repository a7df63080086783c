# MOD A/B: C4 job with each library (SDB_LIB), the eager per-phase breakdown; MOD tests with the last one
for lib in "$@"; do
  echo "== $lib"
  SDB_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err || tail -3 gpurun_out/bench_ab.err
  python tools/show_bench.py gpurun_out/bench_ab.json | grep -E "ms/step|mod_update|certify"
done
timeout 900 python -m pytest tests/test_gpu_mod_train.py -x -q > gpurun_out/t_mod.log 2>&1; echo modtests rc=$?; tail -2 gpurun_out/t_mod.log
