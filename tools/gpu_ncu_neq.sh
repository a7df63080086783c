timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_normal_eq_w -s 1 -c 1 -o gpurun_out/prof_neq python tools/cert_probe.py > gpurun_out/ncu_neq.log 2>&1; echo ncu rc=$?
