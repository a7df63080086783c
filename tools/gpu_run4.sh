timeout 900 python tools/parity_trace.py c4 10 c3 17 c2 9 > gpurun_out/trace2.jsonl 2> gpurun_out/trace2.err
python tools/ref_suite.py run > gpurun_out/ref_suite_rc.txt 2>&1
