"""Quick timing of one config on the GPU (development aid, not the bench contract): graph-replayed
P-ERK steps timed with CUDA events (L2 flushed), single-rate comparison, per-kernel eager profile."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2403_05144_b200 import Perk  # noqa: E402


def timed(p, U, dt, K=20, Wm=5):
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(Wm):
        p.step(U, dt)
    torch.cuda.synchronize()
    ts = []
    s = torch.cuda.current_stream()
    for _ in range(K):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        p.step(U, dt)
        b.record(s)
        ts.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ts]))


def main():
    cfgs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3").split(",")]
    for cfg in cfgs:
        w = W.make(cfg)
        p = Perk(w.problem, w.level_map, w.S, w.E)
        U = p.initial_state(w.ic)
        ms = timed(p, U, w.dt)
        ev = int(p.count_active("elements").sum())
        sr = Perk(w.problem, w.level_map, w.S, [w.S])
        Us = sr.initial_state(w.ic)
        ms_sr = timed(sr, Us, w.dt)
        prof = np.zeros(7)
        for k in [0, 1, 4, 5]:
            if k >= 4 and w.problem["equation"] != "navier_stokes":
                continue
            prof[k] = 3 * p.time_kernels(U.clone(), w.dt, [k], reps=10)
        print(json.dumps({"cfg": cfg, "cells": p.n_cells, "ms_per_step": round(ms, 4),
                          "elem_rhs_per_s": round(ev / ms * 1e3), "single_rate_ms": round(ms_sr, 4),
                          "speedup": round(ms_sr / ms, 3),
                          "graph_ms": {"surf": round(prof[0] / 3, 4), "vol": round(prof[1] / 3, 4),
                                       "br1_traces": round(prof[4] / 3, 4), "br1_grad": round(prof[5] / 3, 4)}}))
        p.close()
        sr.close()


if __name__ == "__main__":
    main()
