"""Full-run parity of the CUDA path against the oracle (BASELINE.json north_star: "within 1e-10 max
relative fp64 state error per conserved variable after the full run"), one process per config so the
single-threaded oracle runs use several host cores.  Step counts: the BASELINE ones for cfg 1-3, and
by default bounded samples for cfg 4 (200 of 2000 steps, 40 device re-meshes) and cfg 5 (20 of 200
steps), whose full oracle runs take hours on one core ("cfg:steps" overrides, e.g. "5:200").  With
ORACLE_OMP=1 the oracle is the OpenMP build (bitwise identical to the serial one; OMP_NUM_THREADS per
process), which makes the full cfg 4 / cfg 5 runs fit one GPU call.  Prints one JSON object;
development / evidence tool, not part of the test suite."""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

PLAN = {1: None, 2: None, 3: None, 4: 200, 5: 20}   # None = the BASELINE step count


def run(arg):
    cfg, steps_override, variant = arg
    import numpy as np
    import torch
    import workloads as W
    from oracle import oracle as O
    from oracle import tableau as T
    from gpu_util import compare_mesh, gpu_state_numpy, rel_err_per_var
    from paper_2403_05144_b200 import Perk
    w = W.make(cfg)
    steps = steps_override or PLAN[cfg] or w.steps
    # variants: p3 = the P-ERK3 family with the config's S, E (f1); alt / early = stage
    # patterns (f2); sc = subcell shock capturing on the contact-band input (f3); i = cfg 4 with the
    # device AMR indicator + controller instead of the seeded map sequence (f3)
    family = pattern = None
    if variant == "p3":
        from workloads import perk3 as P3
        family = fam = P3.family3(w.S, w.E)
    elif variant in ("alt", "early"):
        pattern = {"alt": "alternating", "early": "early"}[variant]
        fam = T.family(w.S, w.E, w.alpha_rule, pattern=pattern)
    else:
        fam = T.family(w.S, w.E, w.alpha_rule)
    if variant == "sc":
        w.problem = dict(w.problem, shock_capturing=W.configs.SHOCK_CAPTURING)
        w.ic = W.configs.contact_band(w.ic)
    ora = O.OracleMesh(w.problem, w.level_map, fam)
    gpu = Perk(w.problem, w.level_map, w.S, w.E, family=family, pattern=pattern)
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    t0 = time.time()
    remeshes = 0
    map_diffs = 0
    if w.remesh_every:
        done = 0
        k = 0
        while done < steps:
            n = min(w.remesh_every, steps - done)
            ora.step(Uo, w.dt, n)
            gpu.step(Ug, w.dt, n)
            done += n
            if done % w.remesh_every == 0 and done < steps:
                k += 1
                if variant == "i":   # indicator-driven AMR (f3): each side adapts with its own controller
                    lm = ora.amr_adapt(Uo, w.meta["amr"])
                    lm_g = gpu.amr_adapt(Ug, w.meta["amr"]).cpu().numpy()
                    map_diffs += int(not np.array_equal(lm, lm_g))
                else:
                    lm = lm_g = w.level_map_seq(k)
                new = O.OracleMesh(w.problem, lm, fam)
                Uo = O.transfer(ora, new, Uo)
                ora = new
                gpu.repartition(lm_g, Ug)
                remeshes += 1
    else:
        ora.step(Uo, w.dt, steps)
        gpu.step(Ug, w.dt, steps)
    torch.cuda.synchronize()
    gpu.sync()
    err = rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo)
    lo, lg = ora.leaves(), gpu.leaves()
    same_mesh = all(np.array_equal(lo[q], lg[q]) for q in ("fx", "fy", "level", "member"))
    try:                                   # faces, per-member lists and stage prefix tables, bitwise
        compare_mesh(ora, gpu)
        same_lists = True
    except AssertionError:
        same_lists = False
    res = {"workload": w.name + (f"_{variant}" if variant else ""), "steps": steps, "baseline_steps": w.steps, "re_meshes": remeshes,
           "cells": int(ora.n), "max_rel_err_per_var": [float(x) for x in err], "mesh_identical": same_mesh,
           "lists_identical": same_lists,
           "pass": bool(err.max() <= 1e-10 and same_mesh and same_lists and map_diffs == 0), "oracle_seconds": round(time.time() - t0, 1)}
    if variant == "i":
        res["amr_maps_differing"] = map_diffs   # near-threshold ties; 0 = every adapted map bit-exact
    out = os.path.join(ROOT, "gpurun_out")                # each config's result as soon as it is done
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, f"full_run_parity_cfg{cfg}{variant}_{steps}.json"), "w") as f:
        json.dump(res, f, indent=1)
    return f"cfg{cfg}{variant}", res


if __name__ == "__main__":
    # argument: comma list of configs, each optionally "cfg[variant]:steps" (e.g. "4:1000,5:200,3p3:500")
    items = [x for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4,5").split(",") if x]
    args = []
    for x in items:
        head, steps = (x.split(":")[0], int(x.split(":")[1])) if ":" in x else (x, None)
        args.append((int(head[0]), steps, head[1:]))
    ctx = mp.get_context("spawn")
    with ctx.Pool(len(args)) as pool:
        res = dict(pool.map(run, args))
    print(json.dumps({"tolerance": 1e-10, "configs": res}, indent=1))
