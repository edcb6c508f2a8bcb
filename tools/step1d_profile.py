"""cfg 1 multirate vs single-rate k_step1d (development aid): a few graph-replayed steps of each, for
ncu (-k regex:k_step1d) or plain event timing.  python tools/step1d_profile.py [steps]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2403_05144_b200 import Perk  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = W.make(1)
out = {}
for name, E in (("multirate", w.E), ("single_rate", [w.S])):
    p = Perk(w.problem, w.level_map, w.S, E)
    U = p.initial_state(w.ic)
    for _ in range(2):
        p.step(U, w.dt)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        p.step(U, w.dt)
    b.record(s)
    torch.cuda.synchronize()
    out[name] = a.elapsed_time(b) / K
    p.close()
print(json.dumps(out))
