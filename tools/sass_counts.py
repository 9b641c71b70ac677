"""Opcode counts of the hot kernels in the built libcosched.so (cuobjdump -sass):
evidence that the scorers issue FADD2 / FMNMX3 / IMAD on TMA-staged (UBLKCP,
SYNCS mbarrier) operands without register spills (STL / LDL).
usage: python tools/sass_counts.py [lib] > profiles/r02/sass_opcodes.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2405_03838_b200/libcosched.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
WANT = ["k_score_pairs_tiledILi2ELi4ELb0", "k_score_pairs_tiledILi2ELi4ELb1", "k_score_pairs_tiledILi2ELi1ELb0",
        "k_score_triples_tiledILi2", "k_pairs_merge_finish", "k_rescore_setsILi2", "k_greedy_scanILi2",
        "k_keys_in_rangeILi2", "k_project_allILi2", "k_gather_fastILi2"]
OPS = ["FADD2", "FADD", "FMNMX3", "FMNMX", "IMAD", "FFMA", "FSETP", "LDS", "STS", "LDG", "STG", "UBLKCP",
       "SYNCS", "BAR", "ATOMG", "RED", "STL", "LDL"]
funcs = re.split(r"\n\s*Function : ", sass)
print(f"# {lib}: static SASS instruction counts per kernel (cuobjdump -sass), sm_100a")
print("# kernel".ljust(46) + "".join(o.rjust(8) for o in OPS))
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    tag = next((w for w in WANT if w in name), None)
    if not tag:
        continue
    cnt = collections.Counter()
    for line in f.split("\n"):
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(?:\.[\w.]+)?", line)
        if m:
            op = m.group(1)
            cnt[op] += 1
    print(tag.ljust(46) + "".join(str(cnt.get(o, 0)).rjust(8) for o in OPS))
