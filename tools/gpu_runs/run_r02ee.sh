mkdir -p gpurun_out/r02ee
O=gpurun_out/r02ee
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-hill --calib-coruns 0 --alloc-k 0 --shard-ws "" > $O/torchrun.json 2> $O/torchrun.err
tail -2 $O/smoke.txt; tail -c 300 $O/torchrun.json; tail -3 $O/torchrun.err
