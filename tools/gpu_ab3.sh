SDB_OMP_TC_CLEN=246 timeout 600 python tools/omp_tc_ab.py tools/_ab/libsdb200_base.so paper_1403_4781_b200/libsdb200.so > gpurun_out/ab246.log 2>&1; echo ab rc=$?
SDB_OMP_TC_CLEN=250 timeout 600 python tools/omp_tc_ab.py tools/_ab/libsdb200_base.so paper_1403_4781_b200/libsdb200.so > gpurun_out/ab250.log 2>&1; echo ab rc=$?
SDB_OMP_TC_CLEN=7 timeout 600 python tools/omp_tc_ab.py tools/_ab/libsdb200_base.so paper_1403_4781_b200/libsdb200.so > gpurun_out/ab7.log 2>&1; echo ab rc=$?
