"""bench.py -- P-ERK multirate DGSEM step on B200 (BASELINE.json metric), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

Workload (default): BASELINE.json configs[2] = cfg 3, 2D Euler on the seeded 3-level quadtree
(62,932 cells, 1.007M nodes), P-ERK2 {4, 8, 16}; DESIGN.md §6 says why cfg 3 is the headline.
A "step" is one full P-ERK step (S = 16 stages: surface-flux + volume/stage kernels per stage).
`value` = element-RHS evaluations/s (sum_r E_r N_C(r) per step / device time per step), whole job.
Timing: W warm-up steps, then K steps each bracketed by CUDA events on the launching stream with
an L2 flush (256 MB write) between timed steps; barrier + synchronize on both sides; max over
ranks.  N > 1 runs independent replicas of the workload (weak scaling; no data-path collective:
the multi-GPU domain decomposition of SURVEY §8(e) is not built).
`other_configs` adds the same measurement for BASELINE cfg 1, 2 (1D, launch-latency bound), cfg 4
(dynamic AMR: device re-mesh every 5 steps inside the timed steps, repartition time reported
separately), cfg 5 (Navier-Stokes, BR1) and cfg 3 with the third-order P-ERK3 family (SURVEY §8(f)
f1), cfg 4 with indicator-driven AMR instead of the seeded map sequence (`4i`: perk_amr_adapt +
perk_repartition every 5 steps) and cfg 3 with the alternating / early-shared stage
patterns (`3alt`, `3early`) and cfg 3 / 5 with subcell shock capturing on a contact
band (`3sc`, `5sc`), so one run shows every config (--extra none skips them).
--impl reference times the oracle (oracle/, plain C, 1 host core) on a bounded sample of the same
workload (full-mesh P-ERK steps, at most ~120 s of CPU work).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "element-RHS evals/s per P-ERK step (fp64)"
UNIT = "element-RHS/s"

# Executed fp64 work of the hot kernels per element-RHS: counted with ncu
# (smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum over all 32 launches of one cfg-3
# step, profiles/r01_fp64_ops_dram_per_step_v13.csv) and divided by the step's 713,596 element-RHS;
# flops = 2 DFMA + DMUL + DADD.  Cold-cache DRAM bytes of the same launches (ncu, per launch average)
# give `traffic`.
VOL_FLOPS_PER_ELEMENT_RHS = 6401.9        # k_vol2d (volume + lift + Jacobian + stage epilogue)
SURF_FLOPS_PER_ELEMENT_RHS = 947.3        # k_surf2d (HLL interface / mortar fluxes)
VOL_DRAM_BYTES_PER_LAUNCH = (1335842816.0 + 74005504.0) / 16   # k_vol2d, cold cache (ncu flushes)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            P = json.load(f)
        return P, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def _fp64_peak():
    """Measured fp64 FMA throughput of this GPU (tools/fp64_peak.cu, 8 independent DFMA chains per
    thread, 148 x 8 blocks of 256 threads), else derived from unit counts and the max clock."""
    exe = os.path.join(ROOT, "paper_2403_05144_b200", "lib", "fp64_peak")
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
        d = json.loads(out.strip().splitlines()[-1])
        return float(d["fp64_tflops"]), "measured: tools/fp64_peak.cu DFMA microbenchmark on this GPU"
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "derived: 148 SM x 64 DFMA/clk x 2 x 1965 MHz"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 20 ms during the clock soak (untimed steps
    of the same workload, >= 0.5 s, so the sample count does not depend on K) and the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _volume_bytes_per_step(count_el, S):
    """Algorithmic HBM bytes of the volume/stage kernel per step: per element-stage
    8 B x 64 doubles for each state-sized vector it must touch:
      stage 1           : read U_n, Fs; write K_1                      -> 3 x 512 B
      first active i>1  : read U_n, K_1 (lazy state), Fs; write U^(i+1) -> 4 x 512 B
      later 1 < i < S   : read U^(i), U_n, K_1, Fs; write U^(i+1)      -> 5 x 512 B
      stage S           : read U^(S), U_n, Fs; write U_{n+1}            -> 4 x 512 B"""
    B = 512
    tot = 3 * B * count_el[0]
    for i in range(2, S + 1):
        n = count_el[i - 1]
        newly = n - (count_el[i - 2] if i > 2 else 0)
        if i == S:
            tot += 4 * B * n
        else:
            tot += 4 * B * newly + 5 * B * (n - newly)
    return tot


class _Timer:
    """CUDA-event timing of P-ERK steps on the launching stream, L2 flushed between timed steps."""

    def __init__(self, torch, dev, ws, dist):
        self.torch, self.ws, self.dist = torch, ws, dist
        self.flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        self.stream = torch.cuda.current_stream()

    def steps(self, run_step, K, Wm):
        torch = self.torch
        for s in range(Wm):
            run_step(-1 - s)
        torch.cuda.synchronize()
        if self.ws > 1:
            self.dist.barrier()
        torch.cuda.synchronize()
        evs = []
        for k in range(K):
            self.flush.fill_(1.0)                      # evict L2 between timed steps
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            run_step(k)
            b.record(self.stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        if self.ws > 1:
            self.dist.barrier()
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]


def _max_over_ranks(torch, dist, ws, dev, x):
    """max over ranks of a per-rank device time (the job takes as long as its slowest replica)"""
    if ws == 1:
        return x
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(ws, elem_rhs_per_step, ms_max):
    """whole-job throughput of ws independent replicas: all units processed / the slowest rank's time"""
    return ws * elem_rhs_per_step / (ms_max * 1e-3)


def measure_config(cfg, K, Wm, timer, torch, dist, ws, dev, with_single=True, order=2, amr=False, pattern=None,
                   sc=False):
    """Device time per P-ERK step of BASELINE config `cfg` (and of the single-rate S-stage P-ERK on
    the same mesh); cfg 4 re-meshes on the device every 5 steps inside the timed steps.  order = 3
    runs the P-ERK3 family with the same S and E (workloads/perk3.py).  amr = True
    (cfg 4) replaces the seeded level-map sequence by the device indicator + controller
    (perk_amr_adapt) before each repartition.  sc = True switches on the subcell
    shock capturing and adds a contact band to the IC (workloads.configs)."""
    from paper_2403_05144_b200 import Perk
    w = W.make(cfg)
    if sc:
        w.problem = dict(w.problem, shock_capturing=W.configs.SHOCK_CAPTURING)
        w.ic = W.configs.contact_band(w.ic)
    fam = single_fam = None
    if order == 3:
        from workloads import perk3 as P3
        fam, single_fam = P3.family3(w.S, w.E), P3.family3(w.S, [w.S])
    perk = Perk(w.problem, w.level_map, w.S, w.E, family=fam, pattern=pattern)
    U = perk.initial_state(w.ic)
    res = {"workload": w.name + ("_perk3" if order == 3 else "") + ("_amr_" + w.meta["amr"]["indicator"] if amr else "")
           + ("_" + pattern if pattern else "") + ("_shock_capturing" if sc else ""),
           "cells": perk.n_cells, "S": w.S, "E": w.E, "order": order, "dt": w.dt}
    if pattern:
        res["pattern"] = pattern
    if amr:
        res["amr"] = w.meta["amr"]
    maps = []
    lm_buf = torch.zeros(w.level_map.shape, dtype=torch.uint8, device=dev)
    if w.remesh_every and not amr:
        # level maps of the re-meshes inside the measured window, uploaded before the timed region
        nmaps = (K + Wm) // w.remesh_every + 1
        maps = [torch.from_numpy(np.ascontiguousarray(w.level_map_seq(k))).to(dev) for k in range(1, nmaps + 1)]

    def timed(p, Ux, Kx):
        """mean ms per step; with re-meshing, the device repartition every remesh_every steps is inside
        the timed steps and timed separately as well"""
        if not w.remesh_every:
            return float(np.mean(timer.steps(lambda k: p.step(Ux, w.dt), Kx, Wm))), []
        state = {"n": 0, "k": 0}
        rp_ev, ad_ev = [], []

        def run_step(_):
            p.step(Ux, w.dt)
            state["n"] += 1
            if state["n"] % w.remesh_every == 0 and (amr or state["k"] < len(maps)):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                if amr:
                    c = torch.cuda.Event(enable_timing=True)
                    c.record(timer.stream)
                    p.amr_adapt(Ux, w.meta["amr"], out=lm_buf)
                    a.record(timer.stream)
                    p.repartition(lm_buf, Ux)
                    ad_ev.append((c, a))
                else:
                    a.record(timer.stream)
                    p.repartition(maps[state["k"]], Ux)
                b.record(timer.stream)
                rp_ev.append((a, b))
                state["k"] += 1
        t = timer.steps(run_step, Kx, Wm)
        torch.cuda.synchronize()
        p.sync()
        timed.adapt_ms = [a.elapsed_time(b) for a, b in ad_ev]
        return float(np.mean(t)), [a.elapsed_time(b) for a, b in rp_ev]

    ms_raw, remesh = timed(perk, U, K)
    if w.remesh_every:
        res["remesh_every"] = w.remesh_every
        res["repartitions_in_run"] = len(remesh)
        res["repartition_ms_mean"] = round(float(np.mean(remesh)), 5) if remesh else None
        if amr:
            res["amr_adapt_ms_mean"] = round(float(np.mean(timed.adapt_ms)), 5) if timed.adapt_ms else None
            res["amr_launches_per_adapt"] = perk.amr_launches()
        ev, st = perk.counters()
        elem_rhs_per_step = ev / max(st, 1)
    else:
        # sum_r E_r N_C(r) from the device counter (the per-stage launch sizes over-count members that
        # do not evaluate a stage under non-standard stage patterns)
        ev, st = perk.counters()
        elem_rhs_per_step = int(round(ev / max(st, 1)))
    ms = _max_over_ranks(torch, dist, ws, dev, ms_raw)
    res.update(ms_per_step=round(ms, 5), element_rhs_per_step=round(float(elem_rhs_per_step), 1),
               value=round(replica_value(ws, elem_rhs_per_step, ms), 1), n_cells_now=perk.n_cells)
    if with_single:
        # single-rate S-stage P-ERK on the same mesh (and the same re-mesh sequence)
        single = Perk(w.problem, w.level_map, w.S, [w.S], family=single_fam,
                      max_cells=w.problem["max_cells"])
        Us = single.initial_state(w.ic)
        ms_s = _max_over_ranks(torch, dist, ws, dev, timed(single, Us, max(3, K // 2) if not w.remesh_every else K)[0])
        if w.remesh_every:
            ev_s, st_s = single.counters()
            cells_per_step = ev_s / max(st_s, 1) / w.S       # mean cell count over the run
        else:
            cells_per_step = perk.n_cells
        single.close()
        res["single_rate_ms_per_step"] = round(ms_s, 5)
        res["multirate_speedup"] = round(ms_s / ms, 4)
        res["ideal_multirate_speedup"] = round(w.S * cells_per_step / elem_rhs_per_step, 4)
    return perk, U, w, res


def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    timer = _Timer(torch, dev, ws, dist)
    fp64_peak, fp64_src = _fp64_peak()

    from paper_2403_05144_b200 import Perk  # noqa: F401  (fails loudly without the CUDA library)
    with ClockSampler(local) as clk:
        w0 = W.make(args.config)
        # clock soak: untimed steps of the headline workload under load (>= 0.5 s)
        from paper_2403_05144_b200 import Perk as _P
        soak = _P(w0.problem, w0.level_map, w0.S, w0.E)
        Usoak = soak.initial_state(w0.ic)
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 0.5:
            for _ in range(50):
                soak.step(Usoak, w0.dt)
            torch.cuda.synchronize()
        soak.close()
        del Usoak
        perk, U, w, res = measure_config(args.config, args.steps, args.warmup, timer, torch, dist, ws, dev)
    n = perk.n_cells
    npe = 4 ** w.problem["dim"]
    ms = res["ms_per_step"]
    value = res["value"]
    elem_rhs_per_step = res["element_rhs_per_step"]
    count_el = [int(x) for x in perk.count_active("elements")]

    # per-kernel device time: CUDA events around graph replays that contain only that kernel kind's
    # launches of a step, launched exactly as perk_step launches them (perk_time_kernels); the eager
    # numbers (events around every individual launch) include ~5 us of launch path per kernel
    from paper_2403_05144_b200.perk import NKINDS
    prof_steps = 3
    ms_e = np.zeros(NKINDS)
    U0 = perk.initial_state(w.ic)
    Up = U0.clone()
    for _ in range(prof_steps):
        m_, _l = perk.profile_step(Up, w.dt)
        ms_e += np.array(m_)
    ms_e /= prof_steps
    kinds = [0, 1] + ([4, 5] if w.problem["equation"] == "navier_stokes" else [])
    ms_k = np.zeros(NKINDS)
    for k in kinds:
        ms_k[k] = perk.time_kernels(U0.clone(), w.dt, [k], reps=10)
    ms_all = perk.time_kernels(U0.clone(), w.dt, kinds, reps=10)
    kern = {"surface": round(ms_k[0], 5), "volume_stage": round(ms_k[1], 5), "all_kinds_graph": round(ms_all, 5),
            "eager_launches": {"surface": round(ms_e[0], 5), "volume_stage": round(ms_e[1], 5)}}
    if w.problem["equation"] == "navier_stokes":
        kern.update(br1_gradient_traces=round(ms_k[4], 5), br1_gradients=round(ms_k[5], 5))
    vol_ms = ms_k[1]
    peaks, src = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    line_roof = None
    if w.problem["dim"] == 2 and w.problem["equation"] == "euler":
        vol_bytes = _volume_bytes_per_step(count_el, w.S)
        launches = w.S
        achieved_gbs = vol_bytes / (vol_ms * 1e-3) / 1e9
        achieved_tf = elem_rhs_per_step * VOL_FLOPS_PER_ELEMENT_RHS / (vol_ms * 1e-3) / 1e12
        kname = "k_vol2d<MODE_STAGE> (volume + surface lift + Jacobian + stage epilogue)"
        roof_hbm = {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(achieved_gbs / hbm, 4), "traffic": round(VOL_DRAM_BYTES_PER_LAUNCH),
                    "kernel": kname, "peak_source": src,
                    "algorithmic_bytes_per_launch": round(vol_bytes / launches),
                    "kernel_ms_per_launch": round(vol_ms / launches, 5),
                    "traffic_note": "ncu dram bytes per launch, cold cache (ncu flushes caches between replays)"}
        roof_alu = {"bound": "alu", "achieved": round(achieved_tf, 3), "peak": round(fp64_peak, 2),
                    "unit": "TFLOP/s", "frac": round(achieved_tf / fp64_peak, 4), "traffic": roof_hbm["traffic"],
                    "kernel": kname, "peak_source": fp64_src,
                    "flops_per_element_rhs": VOL_FLOPS_PER_ELEMENT_RHS}
        roof = roof_alu if roof_alu["frac"] >= roof_hbm["frac"] else roof_hbm
        line_roof = (roof, roof_hbm if roof is roof_alu else roof_alu)

    # end to end through the public API with HOST buffers (pinned), copies inside the timed region
    Uh = U0[:n].cpu().pin_memory()
    e2e_steps = max(3, min(args.steps, 20))
    perk.run_host(Uh, w.dt, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        perk.run_host(Uh, w.dt, 1)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e_val = ws * elem_rhs_per_step / e2e_s
    h2d = int(n * w.nv * npe * 8)
    launches = perk.launches_per_step()
    perk.close()

    others = {}
    if args.extra != "none":
        for item in [x for x in args.extra.split(",") if x]:
            amr = item.endswith("i")
            sc = item.endswith("sc")
            pattern = {"alt": "alternating", "early": "early"}.get(item.lstrip("0123456789"))
            c, order = (int(item[:-2]), 3) if item.endswith("p3") else (int(item.rstrip("ialterysc")), 2)
            if c == args.config and order == 2 and not amr and not pattern and not sc:
                continue
            try:
                p2, _U, _w, r2 = measure_config(c, max(5, min(args.steps, 20)), args.warmup, timer, torch, dist,
                                                 ws, dev, order=order, amr=amr, pattern=pattern, sc=sc)
                r2["dof_stage_updates_per_s"] = round(r2["value"] * 4 ** _w.problem["dim"], 1)
                r2["gpu_launches_per_step"] = p2.launches_per_step()
                p2.close()
                others[f"cfg{item}"] = r2
            except Exception as ex:       # report, do not hide: the line records the failure
                others[f"cfg{item}"] = {"error": repr(ex)[:200]}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, budget_s=args.cpu_budget)

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator workloads/, DESIGN.md §3)",
            "config": {"workload": w.name, "cells": n, "nodes": n * npe, "S": w.S, "E": w.E,
                       "element_rhs_per_step": elem_rhs_per_step, "dt": w.dt,
                       "l2": "flushed between timed steps (256 MB write, outside the events)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
            "dof_stage_updates_per_s": round(value * npe, 1),
            "scalar_dof_stage_updates_per_s": round(value * npe * w.nv, 1),
            "single_rate_ms_per_step": res.get("single_rate_ms_per_step"),
            "multirate_speedup": res.get("multirate_speedup"),
            "ideal_multirate_speedup": res.get("ideal_multirate_speedup"),
            "kernel_ms_per_step": kern,
            "e2e": {"value": round(e2e_val, 1), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d},
            "gpu_launches": launches * args.steps,
            "clocks": clocks,
        }
        if line_roof:
            line["roofline"], line["roofline_other"] = line_roof
        if others:
            line["other_configs"] = others
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def cpu_baseline(w, budget_s=20.0):
    """The oracle as it stands (plain C, single thread) on a bounded sample: whole P-ERK steps of the
    same mesh, as many as fit in ~budget_s (at least one)."""
    from oracle import oracle as O
    from oracle import tableau as T
    fam = T.family(w.S, w.E, w.alpha_rule)
    m = O.OracleMesh(w.problem, w.level_map, fam)
    U = m.initial_state(w.ic)
    t0 = time.perf_counter()
    ev = m.step(U, w.dt, 1)
    dt1 = time.perf_counter() - t0
    k = max(0, int(budget_s / max(dt1, 1e-9)) - 1)
    t1 = time.perf_counter()
    ev2 = m.step(U, w.dt, k) if k > 0 else 0
    dt2 = time.perf_counter() - t1
    total_ev, total_t = (ev2, dt2) if k > 0 else (ev, dt1)
    return {"value": round(total_ev / total_t, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{k if k > 0 else 1} full P-ERK step(s) of {w.name} ({m.n} cells), restricted mode, 1 thread",
            "seconds": round(total_t, 2)}


def run_profile_only(args):
    import torch
    from paper_2403_05144_b200 import Perk
    w = W.make(args.config)
    perk = Perk(w.problem, w.level_map, w.S, w.E)
    U = perk.initial_state(w.ic)
    for _ in range(args.warmup + args.steps):
        perk.step(U, w.dt)
    torch.cuda.synchronize()
    perk.sync()
    print(json.dumps({"profile_only": w.name, "steps": args.warmup + args.steps,
                      "launches_per_step": perk.launches_per_step()}))


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    w = W.make(args.config)
    from oracle import oracle as O
    from oracle import tableau as T
    fam = T.family(w.S, w.E, w.alpha_rule)
    m = O.OracleMesh(w.problem, w.level_map, fam)
    U = m.initial_state(w.ic)
    Wm = max(1, min(args.warmup, 3))               # warm-up steps (no JIT; the last one sizes the sample)
    for _ in range(Wm):
        t0 = time.perf_counter()
        ev = m.step(U, w.dt, 1)
        t_step = time.perf_counter() - t0
    K = max(1, min(args.steps, int(120.0 / max(t_step, 1e-9))))
    t1 = time.perf_counter()
    tot = m.step(U, w.dt, K)
    dt = time.perf_counter() - t1
    value = tot / dt
    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws, "steps": K,
            "warmup": Wm, "ms_per_step": round(1e3 * dt / K, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator workloads/)",
            "config": {"workload": w.name, "cells": m.n, "element_rhs_per_step": int(ev)},
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{K} full P-ERK step(s) of {w.name}, restricted mode, 1 thread "
                                       f"(requested --steps {args.steps}, capped at ~120 s)"},
            "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--extra", default="1,2,4,4i,5,3p3,3alt,3early,3sc,5sc",
                    help="other BASELINE configs measured into other_configs (comma list, 'Np3' = config N "
                         "with the P-ERK3 family, 'Ni' = config N with indicator-driven AMR, "
                         "'Nalt' / 'Nearly' = config N with the alternating / early-shared stage pattern, or 'none')")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true",
                    help="build the workload and run warmup+steps P-ERK steps only (short ncu target)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.profile_only:
        run_profile_only(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
