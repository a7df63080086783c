timeout 300 python tools/omp_tc_probe.py 256 15625 512 8 64 omp_tc 2>&1 | tail -1
for c in 250 8; do echo "clen $c"; SDB_OMP_TC_CLEN=$c timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/bench_clen$c.json 2> gpurun_out/bench_clen$c.err; done
