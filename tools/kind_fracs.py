"""Per-kernel-kind HBM fractions of workload variants (development aid): flushed per-kind graph
replays (perk_time_kernels_ex) against bench.py's algorithmic bytes.
  python tools/kind_fracs.py 5,5e,3,3big     (5e = the cfg-5 mesh and IC with the Euler equations,
  3big = cfg 3 on a 256^2 base grid: 4x the cells, beyond L2)"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_2403_05144_b200 import Perk  # noqa: E402


def variant(name):
    if name == "5e":
        w = W.make(5)
        w.problem = dict(w.problem, equation="euler")
        return w
    if name == "3big":
        return W.make(3, n_base=256)
    return W.make(int(name))


def main():
    names = (sys.argv[1] if len(sys.argv) > 1 else "5,5e").split(",")
    P = bench._peaks()[0]
    hbm = float(P.get("hbm_gbs", P.get("hbm_copy_gbs", 6549.8)))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for name in names:
        w = variant(name)
        p = Perk(w.problem, w.level_map, w.S, w.E)
        U = p.initial_state(w.ic)
        ns = w.problem["equation"] == "navier_stokes"
        kinds = [0, 1] + (([5] if bench.br1_fused() else [4, 5]) if ns else [])
        nb = bench.kernel_bytes_per_step(p, w)
        out = {"variant": name, "cells": p.n_cells}
        for k in kinds:
            ms = p.time_kernels(U.clone(), w.dt, [k], reps=10, flush=flush)
            kn = bench.KIND_NAMES[k]
            out[kn] = {"ms": round(ms, 4), "GBps": round(nb[kn] / ms / 1e6, 1),
                       "frac": round(nb[kn] / ms / 1e6 / hbm, 3)}
        print(json.dumps(out), flush=True)
        p.close()


if __name__ == "__main__":
    main()
