"""Summarise an `ncu --set full` capture into the JSON kept under profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> <out.json> [--kernel REGEX] [--source "how it was captured"]

Writes, per captured launch (the first matching one by default), the duration,
launch shape, occupancy, issue and pipe utilisation, shared-memory wavefronts,
DRAM bytes (traffic_bytes_per_launch = read + write, used by bench.py's
roofline.traffic) and the warp-stall breakdown.
"""
import argparse
import csv
import io
import json
import re
import subprocess

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum",
]
STALL_RE = re.compile(r"^smsp__pcsamp_warps_issue_stalled_(\w+)$")


def _bytes(value: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(value.replace(",", "")) * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    pick = None
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if a.kernel is None or re.search(a.kernel, d.get("Kernel Name", "")):
            pick = r
            break
    if pick is None:
        raise SystemExit("no matching launch")
    d = dict(zip(hdr, pick))
    u = dict(zip(hdr, units))
    out = {"Kernel Name": d["Kernel Name"]}
    for k in KEYS:
        if k in d:
            out[k] = d[k]
    traffic = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in d:
            traffic += _bytes(d[k], u.get(k, "byte"))
            out[k + " [bytes]"] = _bytes(d[k], u.get(k, "byte"))
    stalls = {}
    for k, v in d.items():
        m = STALL_RE.match(k)
        if m and not k.endswith("_not_issued"):
            try:
                stalls[m.group(1)] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    out["stall_breakdown_pct"] = {k: round(100 * v / tot, 1)
                                  for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if 100 * v / tot >= 1.0}
    out["traffic_bytes_per_launch"] = traffic
    out["source"] = a.source
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
