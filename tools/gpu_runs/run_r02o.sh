mkdir -p gpurun_out/r02o
O=gpurun_out/r02o
for i in 1 2; do
  echo "== split $i" >> $O/lb.txt
  timeout 600 python -m pytest tests/test_gpu_loopback.py -q -x -k "8" >> $O/lb.txt 2>&1
  echo "== nosplit $i" >> $O/lb.txt
  COSCHED_SPLIT_GATHER=0 timeout 600 python -m pytest tests/test_gpu_loopback.py -q -x -k "8" >> $O/lb.txt 2>&1
done
echo "== nopdl" >> $O/lb.txt
COSCHED_PDL=0 timeout 600 python -m pytest tests/test_gpu_loopback.py -q -x -k "8" >> $O/lb.txt 2>&1
grep "==\|passed\|failed\|Error" $O/lb.txt
