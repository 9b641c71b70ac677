mkdir -p gpurun_out/r02ff
O=gpurun_out/r02ff
B="--steps 10 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws 8"
for i in 1 2; do
  timeout 300 python bench.py $B > $O/base_$i.json 2>/dev/null
  COSCHED_LIB_PATH=tools/variants/tileend.so timeout 300 python bench.py $B > $O/owner_$i.json 2>/dev/null
done
COSCHED_LIB_PATH=tools/variants/tileend.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exactness.py -q -x > $O/tests.txt 2>&1
python -c "
import json
for f in ['base_1','owner_1','base_2','owner_2']:
    d=json.loads(open('$O/'+f+'.json').read().strip().splitlines()[-1]); print(f, round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), round(d['shard_projection']['per_w']['8']['projected_speedup'],3))
"
tail -2 $O/tests.txt
