"""A/B of library builds on one box (development aid): per kernel kind the flushed graph-replay time
(perk_time_kernels_ex, L2 flushed before each replay) and the flushed step time, each library in its
own process, alternating for several rounds; prints the per-variant median over rounds.
  python tools/ab_kinds.py 5,3 A B [rounds]     (libraries paper_2403_05144_b200/lib/libperk_<X>.so;
  a variant "X:NAME=VALUE" runs library X with that environment variable set)"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import workloads as W
from paper_2403_05144_b200 import Perk
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = {{}}
for item in sys.argv[1].split(","):
    cfg = int(item.rstrip("sc"))
    w = W.make(cfg)
    if item.endswith("sc"):
        w.problem = dict(w.problem, shock_capturing=W.configs.SHOCK_CAPTURING)
        w.ic = W.configs.contact_band(w.ic)
    p = Perk(w.problem, w.level_map, w.S, w.E)
    U = p.initial_state(w.ic)
    kinds = [0, 1] + ([4, 5] if w.problem["equation"] == "navier_stokes" else []) + ([6] if item.endswith("sc") else [])
    r = {{k: p.time_kernels(U.clone(), w.dt, [k], reps=20, flush=flush) for k in kinds}}
    for _ in range(5):
        p.step(U, w.dt)
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(30):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); p.step(U, w.dt); b.record(s)
        ts.append((a, b))
    torch.cuda.synchronize()
    r["step"] = float(np.median([a.elapsed_time(b) for a, b in ts]))
    out[item] = r
    p.close()
print(json.dumps(out))
"""


def main():
    cfgs, variants = sys.argv[1], sys.argv[2:]
    rounds = 3
    if variants and variants[-1].isdigit():
        rounds = int(variants.pop())
    res = {v: [] for v in variants}
    for _ in range(rounds):
        for v in variants:
            lib, _, extra = v.partition(":")       # variant "X" or "X:NAME=VALUE" (an environment knob)
            env = dict(os.environ, PERK_LIB_PATH=os.path.join(ROOT, "paper_2403_05144_b200", "lib", f"libperk_{lib}.so"))
            if extra:
                k_, _, v_ = extra.partition("=")
                env[k_] = v_
            o = subprocess.run([sys.executable, "-c", WORKER.format(root=ROOT), cfgs], capture_output=True, text=True,
                               env=env)
            if o.returncode:
                print(v, "failed", o.stderr[-500:])
                continue
            res[v].append(json.loads(o.stdout.strip().splitlines()[-1]))
    summary = {}
    for v, runs in res.items():
        summary[v] = {}
        for cfg in runs[0] if runs else []:
            summary[v][cfg] = {k: round(statistics.median(r[cfg][k] for r in runs), 4) for k in runs[0][cfg]}
    print(json.dumps({"rounds": rounds, "median": summary, "all": res}))


if __name__ == "__main__":
    main()
