#!/bin/bash
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 5000 > gpurun_out/var.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/var.json').read().strip().split('\n')[-1]); print('$v', 'alloc %.2f ms' % d['allocation_ms'], 'rounds', d['allocation_rounds'])"
done
