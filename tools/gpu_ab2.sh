# A/B vs base of the fused OMP + its tests
timeout 600 python tools/omp_tc_ab.py tools/_ab/libsdb200_base.so paper_1403_4781_b200/libsdb200.so > gpurun_out/ab.log 2>&1; echo ab rc=$?
timeout 600 python -m pytest tests/test_gpu_omp_tc.py -q --timeout 600 > gpurun_out/t_omp_tc.log 2>&1; echo tests rc=$?
