timeout 1800 python -m pytest tests -q -m gpu --timeout 1500 -x > gpurun_out/gputest_all.log 2>&1; echo all rc=$?
for t in 4 8 16; do echo "threads $t"; SDB_UPLOAD_THREADS=$t timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(' device', round(d['ms_per_step'],1), 'e2e', round(d['e2e'].get('ms_per_step'),1), 'pageable', round(d.get('e2e_pageable',{}).get('ms_per_step'),1))"; done > gpurun_out/pageable.log 2>&1
