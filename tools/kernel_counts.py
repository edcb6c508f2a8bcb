"""ncu counts per kernel kind of one P-ERK step (bench.py's fp64 flops and `traffic`).

On the GPU box (after the same command ran without ncu):
  ncu --metrics <METRICS> --clock-control none --csv --log-file gpurun_out/counts_cfg5.csv \
      python bench.py --profile-only --config 5 --steps 1 --warmup 3
Here:
  python tools/kernel_counts.py gpurun_out/counts_cfg5.csv 5 4 [gpurun_out/lib_sha16.txt]
writes profiles/r02_kernel_counts_cfg5.json: per kind the executed fp64 flops (2 DFMA + DMUL + DADD,
thread-level SASS counts) and the cold-cache DRAM bytes (ncu flushes caches between replays) summed
over the kind's launches and divided by the number of P-ERK steps the command ran (warmup + steps),
plus the sha256 prefixes of the kernel sources (src_sha16: run this with the sources the GPU-side command
was built from) and of the library that produced them (bench.py marks counts of another build):
the file the GPU-side command wrote (sha256sum of the .so it ran), else the local library.
"""
import collections
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
KINDS = {"k_surf2d": "surface", "k_vol2d": "volume_stage", "k_gsurf2d": "br1_gradient_traces",
         "k_grad2d": "br1_gradients", "k_sc_alpha": "shock_capturing_alpha"}


def parse(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    per_launch = collections.defaultdict(dict)
    names = {}
    for r in rows:
        lid = int(r[0])
        names[lid] = r[4].split("(")[0].replace("void ", "").split("<")[0].strip().split("::")[-1]
        try:
            per_launch[lid][r[-3]] = float(r[-1].replace(",", ""))
        except ValueError:
            pass
    return names, per_launch


def summarise(path, steps):
    names, per_launch = parse(path)
    agg = collections.defaultdict(lambda: collections.Counter())
    for lid, nm in names.items():
        kind = KINDS.get(nm)
        if kind is None:
            continue
        m = per_launch[lid]
        agg[kind]["launches"] += 1
        agg[kind]["dram"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        agg[kind]["flops"] += 2 * m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0) + \
            m.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0) + \
            m.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0)
        agg[kind]["ns"] += m.get("gpu__time_duration.sum", 0.0)
    out = {}
    for kind, c in agg.items():
        out[kind] = {"launches_per_step": c["launches"] / steps, "dram_bytes_per_step": round(c["dram"] / steps),
                     "fp64_flops_per_step": round(c["flops"] / steps),
                     "cold_us_per_step": round(c["ns"] / steps / 1e3, 2)}
    return out


def source_sha16():
    sys.path.insert(0, ROOT)
    from paper_2403_05144_b200.build import source_sha16 as f
    return f()


def lib_sha():
    with open(os.path.join(ROOT, "paper_2403_05144_b200", "lib", "libperk_b200.so"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()[:16]


if __name__ == "__main__":
    src, cfg, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    sha = open(sys.argv[4]).read().split()[0][:16] if len(sys.argv) > 4 else lib_sha()
    res = {"config": cfg, "source": os.path.basename(src), "steps_profiled": steps, "lib_sha16": sha, "src_sha16": source_sha16(),
           "command": f"ncu --metrics {','.join(METRICS)} --clock-control none --csv "
                      f"python bench.py --profile-only --config {cfg} --steps 1 --warmup {steps - 1}",
           "kinds": summarise(src, steps)}
    dst = os.path.join(ROOT, "profiles", f"r02_kernel_counts_cfg{cfg}.json")
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))
