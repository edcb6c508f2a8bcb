"""Cost of the subcell shock capturing (development aid, not the bench contract): cfg 3 / cfg 5 with the
contact-band IC, P-ERK step time with and without shock capturing (CUDA events on the context
stream, L2 flushed between steps), the per-kind split of one eager step, the device time of the
kernel kinds alone (perk_time_kernels: 1 volume, 0 surface, 6 blending factors), and the fraction
of blended elements.  `--ncu`: 3 steps with shock capturing on only (for an ncu launch list / --set full capture)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2403_05144_b200 import Perk  # noqa: E402

KINDS = ["surface", "volume", "mesh", "transfer", "br1_traces", "br1_grad", "sc_alpha"]


def timed_steps(p, U, dt, n, flush):
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(n):
        flush.fill_(1.0)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        p.step(U, dt)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.mean(ts))


def main():
    ncu = "--ncu" in sys.argv
    cfgs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "3,5").split(",")]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    out = {}
    for cfg in cfgs:
        w = W.make(cfg)
        ic = W.configs.contact_band(w.ic)
        res = {}
        for name, sc in [("off", None), ("on", W.configs.SHOCK_CAPTURING),
                         ("alpha_fixed_1", dict(W.configs.SHOCK_CAPTURING, alpha_fixed=1.0))]:
            if ncu and name != "on":
                continue
            prob = dict(w.problem) if sc is None else dict(w.problem, shock_capturing=sc)
            p = Perk(prob, w.level_map, w.S, w.E)
            U = p.initial_state(ic)
            if ncu:
                p.step(U, w.dt, 3)
                torch.cuda.synchronize()
                p.close()
                continue
            p.step(U, w.dt, 3)
            r = {"ms_per_step": round(timed_steps(p, U, w.dt, 10, flush), 5),
                 "launches_per_step": p.launches_per_step()}
            ms, nl = p.profile_step(U, w.dt)
            r["eager_ms_by_kind"] = {KINDS[k]: round(ms[k], 4) for k in range(len(KINDS)) if nl[k]}
            for k, nm in [(1, "volume"), (0, "surface"), (6, "sc_alpha")]:
                if nl[k]:
                    V = U.clone()
                    r[f"alone_ms_{nm}"] = round(p.time_kernels(V, w.dt, [k], reps=5), 5)
            if sc is not None:
                _, a = p.sc_alpha(U)
                a = a.cpu().numpy()
                r["blended_fraction"] = round(float(np.count_nonzero(a)) / len(a), 4)
            torch.cuda.synchronize()
            p.close()
            res[name] = r
        out[f"cfg{cfg}"] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
