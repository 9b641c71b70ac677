mkdir -p gpurun_out/r02x
O=gpurun_out/r02x
for c in 1 2 3 4 6; do
  echo "== chunks $c" >> $O/chunks.txt
  COSCHED_PROJ_CHUNKS=$c timeout 300 python tools/shard_prof.py C4 1 8:7 >> $O/chunks.txt 2>&1
  COSCHED_PROJ_CHUNKS=$c COSCHED_PREP_EVENTS=1 timeout 300 python tools/shard_prof.py C4 1 2> $O/ev_$c.txt > /dev/null
  tail -1 $O/ev_$c.txt >> $O/chunks.txt
done
cat $O/chunks.txt
