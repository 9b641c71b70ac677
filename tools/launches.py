"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel times of one step."""
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    print(f)
    for r in rows[1:]:
        print(f"   {float(r[vi].replace(',', '')) / 1e3:9.2f} us  {r[ki][:90]}")
