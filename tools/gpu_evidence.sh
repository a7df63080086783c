# full default bench (driver contract), reference arm, launch list + ncu of the top kernel
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
python tools/profile_step.py c4 2 > gpurun_out/step_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c4.csv \
    python tools/profile_step.py c4 2 > gpurun_out/ncu_step.log 2>&1; echo launches rc=$?
