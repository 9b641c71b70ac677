mkdir -p gpurun_out/r02bb
O=gpurun_out/r02bb
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
timeout 300 python tools/alloc_prof.py C4 5000 8 | tail -1 > $O/alloc.txt 2>&1
timeout 300 python tools/alloc_prof.py C5 666 5 | tail -1 >> $O/alloc.txt 2>&1
tail -2 $O/pytest.txt; cat $O/alloc.txt
