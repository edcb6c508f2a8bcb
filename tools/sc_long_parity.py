"""Long-run parity of the shock-capturing path (development / evidence tool): cfg-3 structure with
the contact band, P-ERK steps on the device and in the oracle, the relative error per conserved
variable recorded every `every` steps (the Hennemann-Gassner logistic has slope s/T ~ 6.5e3, so
rounding differences in the modal energies are amplified into the blending factor; this shows how
the state difference grows over a run).  Prints one JSON object."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import tableau as T  # noqa: E402
from gpu_util import gpu_state_numpy, rel_err_per_var  # noqa: E402
from paper_2403_05144_b200 import Perk  # noqa: E402


def run(n_base, steps, every):
    w = W.make(3) if n_base is None else W.make(3, n_base=n_base)
    p = dict(w.problem, shock_capturing=W.configs.SHOCK_CAPTURING)
    ic = W.configs.contact_band(w.ic)
    ora = O.OracleMesh(p, w.level_map, T.family(w.S, w.E, w.alpha_rule))
    gpu = Perk(p, w.level_map, w.S, w.E)
    Uo = ora.initial_state(ic)
    Ug = gpu.initial_state(ic)
    hist = []
    done = 0
    while done < steps:
        n = min(every, steps - done)
        ora.step(Uo, w.dt, n)
        gpu.step(Ug, w.dt, n)
        torch.cuda.synchronize()
        done += n
        err = rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo)
        _, a = ora.sc_alpha(Uo)
        hist.append({"step": done, "max_rel_err": float(err.max()), "blended": int(np.count_nonzero(a))})
    return {"cells": int(ora.n), "steps": steps, "history": hist}


if __name__ == "__main__":
    out = {"cfg3_n16": run(16, int(sys.argv[1]) if len(sys.argv) > 1 else 500, 50),
           "cfg3_full": run(None, int(sys.argv[2]) if len(sys.argv) > 2 else 40, 10)}
    print(json.dumps(out, indent=1))
