"""Timing of the device AMR path on cfg 4 (development aid, not the bench contract): perk_amr_adapt
(indicator + controller + balance) and perk_repartition, CUDA events on the context stream, L2 flushed
between repetitions.  `--ncu` runs a few adapts only (for an ncu launch list / --set full capture)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2403_05144_b200 import Perk  # noqa: E402


def main():
    ncu = "--ncu" in sys.argv
    w = W.make(4)
    p = Perk(w.problem, w.level_map, w.S, w.E)
    U = p.initial_state(w.ic)
    lm = torch.zeros(w.level_map.shape, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    out = {"cells": p.n_cells}
    for name, amr in [("enstrophy", w.meta["amr"]),
                      ("hennemann_gassner", dict(indicator="hennemann_gassner", variable="rho_p", base_level=0,
                                                 med_level=2, max_level=4, med_threshold=0.01, max_threshold=0.1)),
                      ("lohner", dict(indicator="lohner", variable="v_x", base_level=0, med_level=2, max_level=4,
                                      med_threshold=0.003, max_threshold=0.03))]:
        reps = 2 if ncu else 20
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
        p.amr_adapt(U, amr, out=lm)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            p.amr_adapt(U, amr, out=lm)
            b.record(s)
            ts.append((a, b))
        torch.cuda.synchronize()
        ti = []
        for _ in range(reps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            p.amr_indicator(U, amr)
            b.record(s)
            ti.append((a, b))
        torch.cuda.synchronize()
        lmn = lm.cpu().numpy().astype(np.float64)
        out[name] = {"adapt_ms_median": float(np.median([a.elapsed_time(b) for a, b in ts])),
                     "indicator_ms_median": float(np.median([a.elapsed_time(b) for a, b in ti])),
                     "cells_after": int((4.0 ** (lmn - w.problem["max_level"])).sum() + 0.5)}
    if not ncu:
        # repartition, ping-pong between the seeded map and the enstrophy-adapted map
        p.amr_adapt(U, w.meta["amr"], out=lm)
        lm0 = torch.from_numpy(np.ascontiguousarray(w.level_map)).cuda()
        tr = []
        for k in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            p.repartition(lm if k % 2 == 0 else lm0, U)
            b.record(s)
            tr.append((a, b))
        torch.cuda.synchronize()
        p.sync()
        out["repartition_ms_median"] = float(np.median([a.elapsed_time(b) for a, b in tr]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
