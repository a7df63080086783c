timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_certify -s 2 -c 1 -o gpurun_out/prof_cert python tools/cert_probe.py > gpurun_out/ncu_cert.log 2>&1; echo ncu rc=$?
