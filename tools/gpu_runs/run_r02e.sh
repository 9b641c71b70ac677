mkdir -p gpurun_out/r02e
O=gpurun_out/r02e
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
B="--steps 10 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0"
timeout 300 python bench.py $B > $O/bench_pdl.json 2> $O/bench_pdl.err
COSCHED_PDL=0 timeout 300 python bench.py $B > $O/bench_nopdl.json 2> $O/bench_nopdl.err
for v in default l2ld l2ldst; do
  if [ $v = default ]; then L=""; else L="COSCHED_LIB_PATH=tools/variants/$v.so"; fi
  env $L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"score_triples_tiled" -c 1 --csv --log-file $O/dram_c5_$v.csv python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws "" > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_greedy_scan -s 20 -c 1 -o $O/scan python tools/alloc_prof.py C4 5000 > $O/scan_ncu.log 2>&1
tail -n 3 $O/pytest.txt
