"""Cost of the domain decomposition (f4) on ONE device: P sub-domains of one mesh held by one process run
their stage kernels and ghost exchanges back to back on one stream, so the step time against the
undecomposed step shows what the decomposition adds (duplicated boundary faces, pack / copy kernels,
2-3 x P launches per stage) -- not a scaling number (this pool leases one GPU).
  python tools/dd_overhead.py [cfg] [P,P,...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2403_05144_b200 import DomainGroup, Perk  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
Ps = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
w = W.make(cfg)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()


def timed(step, n=10, warm=3):
    for _ in range(warm):
        step()
    ts = []
    for _ in range(n):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); step(); b.record(s)
        ts.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ts]))


p = Perk(w.problem, w.level_map, w.S, w.E)
U = p.initial_state(w.ic)
out = {"workload": w.name, "cells": p.n_cells, "undecomposed_ms_per_step": round(timed(lambda: p.step(U, w.dt)), 4)}
p.close()
for P in Ps:
    g = DomainGroup(w.problem, w.level_map, w.S, w.E, P)
    Us = g.initial_state(w.ic)
    out[f"P{P}_ms_per_step_one_device"] = round(timed(lambda: g.step(Us, w.dt)), 4)
    out[f"P{P}_owned_ranges"] = [int(x) for x in np.asarray(g.ranges()).ravel()][: 2 * P]
    g.close()
print(json.dumps(out))
