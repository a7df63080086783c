for g in 4 8 16; do timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra --groups $g > gpurun_out/bench_g$g.json 2> gpurun_out/bench_g$g.err; echo g$g rc=$?; done
