python tools/profile_step.py c2 2 > gpurun_out/step_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c2.csv \
    python tools/profile_step.py c2 2 > gpurun_out/ncu_step.log 2>&1; echo launches rc=$?
