"""Build libperk_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "perk_b200.cu")
OUT = os.path.join(HERE, "lib", "libperk_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-shared", "-Xptxas", "-v"]


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in sorted(os.listdir(d))] + [os.path.join(ROOT, "include", "perk.h")]


def source_sha16() -> str:
    """sha256 prefix of the kernel sources (csrc/, include/perk.h): identifies the code a profile was taken on
    (the .so itself is not bit-reproducible from build to build)."""
    import hashlib
    h = hashlib.sha256()
    for f in sources():
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


TOOLS = [("fp64_peak.cu", "fp64_peak")]   # measured fp64 FMA peak (bench.py roofline denominator)


def build_tools(force: bool = False) -> None:
    for src, exe in TOOLS:
        s = os.path.join(ROOT, "tools", src)
        o = os.path.join(HERE, "lib", exe)
        if force or not os.path.exists(o) or os.path.getmtime(o) < os.path.getmtime(s):
            subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", o, s])


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    newest = max(os.path.getmtime(s) for s in sources())
    build_tools(force)
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= newest:
        return OUT
    cmd = [NVCC] + FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", OUT, SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    with open(os.path.join(HERE, "lib", "ptxas_info.txt"), "w") as f:   # registers / spills / smem per kernel
        f.write("".join(l for l in res.stderr.splitlines(True) if "Compile time" not in l))
    if verbose:
        print(res.stderr)
    return OUT


def build_debug(force: bool = True) -> str:
    """lib/libperk_debug.so: the same library with the device-side bounds checks (PERK_DASSERT) and the
    race-exposure jitter (perk_debug_jitter) on; run the GPU tests against it with
    PERK_LIB_PATH=<that path> (compute-sanitizer is not available on the GPU pool)."""
    out = os.path.join(HERE, "lib", "libperk_debug.so")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(s) for s in sources()):
        return out
    cmd = [NVCC] + [f for f in FLAGS if f not in ("-Xptxas", "-v")] + ["-DPERK_DEBUG", "-I", os.path.join(ROOT, "include"),
                                                                      "-o", out, SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    return out


if __name__ == "__main__":
    import sys
    print(build_debug() if "--debug" in sys.argv else build(force=True))
