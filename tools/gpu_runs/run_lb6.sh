mkdir -p gpurun_out/lb6
export COSCHED_NCCL_LIB=$PWD/tests/loopback/libloopback_nccl.so
python -c "import sys; sys.path.insert(0,'tests'); import loopback; loopback.build()"
for i in 1 2 3 4 5 6; do
  for W in 2 3 8; do
    timeout 300 python tests/loopback_ranks.py $W > gpurun_out/lb6/w${W}_$i.txt 2>&1; echo "W=$W i=$i rc=$?"
  done
done > gpurun_out/lb6/summary.txt
cat gpurun_out/lb6/summary.txt
for f in gpurun_out/lb6/w*.txt; do if grep -q Error $f; then echo $f; grep -E "^case|Error" $f | tail -3; fi; done
