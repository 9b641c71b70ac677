#!/bin/bash
# Run the C4 bench under several env-var variants (scorer only): prints value + scorer ms.
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --alloc-k 0 --no-hill --calib-coruns 0 > gpurun_out/var.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/var.json').read().strip().split('\n')[-1]); print('$v', '%.4g cand/s' % d['value'], 'scorer %.3f ms' % d['roofline']['kernel_ms'], 'frac %.3f' % d['roofline']['frac'])"
done
