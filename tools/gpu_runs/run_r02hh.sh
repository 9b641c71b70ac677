mkdir -p gpurun_out/r02hh
O=gpurun_out/r02hh
for i in 1 2 3; do
  timeout 300 python tools/shard_prof.py C4 1 8:5 8:7 > $O/ev1_$i.txt 2>&1
  COSCHED_NO_EV1=1 timeout 300 python tools/shard_prof.py C4 1 8:5 8:7 > $O/noev1_$i.txt 2>&1
done
for i in 1 2 3; do echo "== ev1 $i"; cat $O/ev1_$i.txt | awk '{print $1,$2,$7}'; echo "== noev1 $i"; cat $O/noev1_$i.txt | awk '{print $1,$2,$7}'; done
