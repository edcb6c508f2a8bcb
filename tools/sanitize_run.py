"""Small end-to-end run of every code path for compute-sanitizer (memcheck / racecheck / initcheck):
cfg 1, 2 (1D, single-CTA step and the two-launch path), cfg 3 structure (2D Euler, mortars), a
non-periodic 2D variant (boundary faces), cfg 5 structure (BR1), rhs_eval with masks, a cfg-4
structure with two device re-meshes and device AMR adaptations (three indicators), stage patterns
(alternating, non-nested), Heun weights, a P-ERK3 family and subcell shock capturing."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2403_05144_b200 import Perk  # noqa: E402


def run(w, steps, problem=None, remesh=False, amr=False, **kw):
    p = Perk(problem or w.problem, w.level_map, w.S, w.E, max_cells=4 * W.configs.count_leaves(w), **kw)
    U = p.initial_state(w.ic)
    p.step(U, w.dt, steps)
    for mask in (1, (1 << len(w.E)) - 1):
        p.rhs(U, mask)
    if remesh:
        for k in (1, 2):
            p.repartition(w.level_map_seq(k), U)
            p.step(U, w.dt, 2)
    if amr:
        for a in (w.meta["amr"],
                  dict(indicator="hennemann_gassner", variable="rho_p", base_level=0, med_level=1, max_level=3,
                       med_threshold=0.01, max_threshold=0.1),
                  dict(indicator="lohner", variable="v_x", base_level=0, med_level=1, max_level=3,
                       med_threshold=0.003, max_threshold=0.03)):
            lm = p.amr_adapt(U, a)
            p.repartition(lm, U)
            p.step(U, w.dt, 2)
    torch.cuda.synchronize()
    p.sync()
    assert torch.isfinite(U[: p.n_cells]).all()
    p.close()


run(W.make(1), 3)
run(W.make(2, n_base=32, w1=8, w2=4), 3)
w3 = W.make(3, n_base=8)
run(w3, 2)
run(w3, 2, problem=dict(w3.problem, periodic=(0, 1), bc_state=(1.0, 1.0, 1.0, 1.0 / 0.4 + 1.0)))
run(W.make(5, n_base=8), 2)
w4 = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
w4.S, w4.E = 16, [4, 6, 10, 16]
run(w4, 2, remesh=True, amr=True)
run(w3, 2, pattern="alternating")
run(w3, 2, pattern=[[1, 5, 9, 16], [1, 2, 4, 6, 8, 10, 12, 16], "standard"], c_S=1.0)
run(W.make(2, n_base=512), 2, pattern="early")
from workloads import perk3 as P3  # noqa: E402
run(w3, 2, family=P3.family3(w3.S, w3.E))
# subcell shock capturing (fused and stand-alone smoothing), Euler + NS, with re-meshes
SC = W.configs.SHOCK_CAPTURING
w3j = W.make(3, n_base=8)
w3j.ic = W.configs.contact_band(w3j.ic)
run(w3j, 2, problem=dict(w3j.problem, shock_capturing=SC))
os.environ["PERK_SC_FUSED"] = "0"
run(w3j, 2, problem=dict(w3j.problem, shock_capturing=SC))
del os.environ["PERK_SC_FUSED"]
w5j = W.make(5, n_base=8)
w5j.ic = W.configs.contact_band(w5j.ic)
run(w5j, 2, problem=dict(w5j.problem, shock_capturing=dict(SC, alpha_fixed=1.0)))
w4.ic = W.configs.contact_band(w4.ic)
run(w4, 2, problem=dict(w4.problem, shock_capturing=SC), remesh=True)
print("sanitize run ok")
