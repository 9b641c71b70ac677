"""Build compile-time variants of libcosched.so for A/B timing on the GPU box
(tools/variants/<name>.so, selected with COSCHED_LIB_PATH). Usage:
python tools/build_variants.py NAME=DEFINE[,DEFINE...] ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_03838_b200 import build  # noqa: E402

out_dir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants")
os.makedirs(out_dir, exist_ok=True)
for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    defines = [d for d in defs.split(",") if d]
    print(build.build(force=True, defines=defines, out=os.path.join(out_dir, name + ".so")))
