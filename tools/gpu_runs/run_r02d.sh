mkdir -p gpurun_out/r02d
O=gpurun_out/r02d
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
COSCHED_LIB_PATH=tools/variants/scanprof.so COSCHED_GREEDY_STATS=1 timeout 300 python tools/alloc_prof.py C4 5000 > $O/scanprof_c4.txt 2>&1
COSCHED_LIB_PATH=tools/variants/scanprof.so COSCHED_GREEDY_STATS=1 timeout 300 python tools/alloc_prof.py C5 666 > $O/scanprof_c5.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"score_(pairs|triples)_tiled" --csv --log-file $O/dram_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws "" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"score_(pairs|triples)_tiled" -c 3 --csv --log-file $O/dram_c5.csv python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws "" > /dev/null 2>&1
tail -n 3 $O/pytest.txt; cat $O/scanprof_c4.txt $O/scanprof_c5.txt
