mkdir -p gpurun_out/r02f
O=gpurun_out/r02f
for v in l2bnd l2bndn; do
  COSCHED_LIB_PATH=tools/variants/$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"score_triples_tiled" -c 1 --csv --log-file $O/dram_c5_$v.csv python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws "" > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_greedy_scan -c 3 -o $O/scan python tools/alloc_prof.py C4 5000 > $O/scan_ncu.log 2>&1
ls $O
