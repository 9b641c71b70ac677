mkdir -p gpurun_out/r02t
O=gpurun_out/r02t
bash tools/sanitize.sh r02t_san > $O/sanitize_summary.txt 2>&1
bash tools/gpu_bench_profile.sh r02t_c4 > $O/prof_c4.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 666 > $O/bench_c5.json 2> $O/bench_c5.err
cat $O/sanitize_summary.txt; tail -c 400 gpurun_out/r02t_c4/bench.json
