"""Build lib/libperk_<NAME>.so with extra -D flags (A/B timing of build variants with tools/ab_kinds.py):
  python tools/build_variant.py NAME [-DMACRO=VALUE ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_05144_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.HERE, "lib", f"libperk_{name}.so")
cmd = [B.NVCC] + B.FLAGS + defs + ["-I", os.path.join(ROOT, "include"), "-o", out, B.SRC]
res = subprocess.run(cmd, capture_output=True, text=True)
if res.returncode != 0:
    sys.exit(res.stdout + res.stderr)
fn, spills = None, []
for l in res.stderr.splitlines():
    if "Compiling entry function" in l:
        fn = l.split("'")[1]
    elif "spill" in l and " 0 bytes spill stores" not in l:
        spills.append((fn, l.strip()))
print(out, "spilling kernels:", len(spills))
for f, l in spills:
    print("  ", f[:90], l)
