"""bench.py -- P-ERK multirate DGSEM step on B200 (BASELINE.json metric), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

Workload (default): BASELINE.json configs[4] = cfg 5, the largest configuration: 2D Navier-Stokes
(BR1) on the seeded 4-level quadtree (305,827 cells, 4.89M nodes), P-ERK2 {4, 8, 16, 32}; DESIGN.md
§6 says why cfg 5 is the headline.  A "step" is one full P-ERK step (S = 32 stages: BR1 gradient
traces + gradients, surface flux, volume/stage kernels per stage).
`value` = element-RHS evaluations/s (sum_r E_r N_C(r) per step / device time per step), whole job.
Timing: W warm-up steps, then K steps each bracketed by CUDA events on the launching stream with
an L2 flush (256 MB write) between timed steps; barrier + synchronize on both sides; max over
ranks.  N > 1 decomposes ONE problem over the N GPUs (E-weighted Morton ranges, per-stage ghost exchange
by NCCL point-to-point; "scaling": "strong"); --replicas runs N independent copies instead.
Per kernel kind: graph replays holding only that kind's launches of a step, L2 flushed between the
replays (perk_time_kernels_ex), against its algorithmic bytes (`kernel_bytes_per_step`)
and, from the committed ncu counts of the same kernels (profiles/r02_kernel_counts_cfg*.json), its
executed fp64 flops; `roofline` is the dominant kernel's, `roofline_kernels` lists every kind.
`other_configs` adds the same measurement for BASELINE cfg 3 (with its own per-kernel rooflines) and
cfg 1, 2 (1D, launch-latency bound), cfg 4 (dynamic AMR: device re-mesh every 5 steps inside the
timed steps, repartition time reported separately), cfg 3 with the third-order P-ERK3 family
(SURVEY §8(f) f1), cfg 4 with indicator-driven AMR instead of the seeded map sequence (`4i`:
perk_amr_adapt + perk_repartition every 5 steps), cfg 3 with the alternating /
early-shared stage patterns (`3alt`, `3early`) and cfg 3 / 5 with subcell shock
capturing on a contact band (`3sc`, `5sc`), so one run shows every config
(--extra none skips them).
cpu_baseline: the oracle (oracle/, plain C) on this host, all cores (OpenMP build, bitwise the
serial one) and 1 thread, on bounded samples of the same workload.
--impl reference times the same oracle on all host cores on a bounded sample (a few minutes at most).
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

# kernel kinds of perk_time_kernels / perk_profile_step (include/perk.h PERK_NUM_KERNEL_KINDS)
KIND_NAMES = {0: "surface", 1: "volume_stage", 4: "br1_gradient_traces", 5: "br1_gradients"}
KERNEL_OF_KIND = {0: "k_surf2d", 1: "k_vol2d", 4: "k_gsurf2d", 5: "k_grad2d"}
LIB = os.path.join(ROOT, "paper_2403_05144_b200", "lib", "libperk_b200.so")


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


def kernel_bytes_per_step(perk, w):
    """Algorithmic HBM bytes per P-ERK step of every 2D kernel kind, from the device
    lists (standard stage pattern, P-ERK2): the bytes each kernel must move at least, counting a
    lazily formed stage state U_n + dt c_i K_1 as two reads.  Units: a state block of an element
    512 B (16 nodes x 4 variables x 8 B), a face trace 128 B (4 nodes x 4 variables), a face-flux
    slot 128 B, a BR1 face slice of Gs / Vt 96 B (4 nodes x 3 components).  Member r (E[r]) is
    active at stage i iff i = 1 or i >= S - E[r] + 2 and its stage state is lazy iff
    2 <= i <= S - E[r] + 2.
      k_vol2d   stage 1: U_n + Fs read, K_1 write; 1 < i < S: (U^(i) or lazy U_n, K_1) + U_n + K_1 +
                Fs read, U^(i+1) write; stage S: state + U_n + Fs read, U_{n+1} write (+ Dv 384 B, NS)
      k_surf2d  interface: 2 traces + 2 flux slots (+ 2 Vt slices, NS); mortar: 3 traces + 3 slots
                (+ 3 Vt slices); boundary: 1 trace + 1 slot
      k_gsurf2d (NS) active + halo interfaces: 2 traces + 2 Gs slices; mortars: 3 traces + 3 slices;
                halo items are lazy (their member is inactive at the stage)
      k_grad2d  (NS) active + halo elements: stage state + Gs (384 B) read, Vt (384 B) write; active
                elements also write their viscous volume term Dv (384 B, read by k_vol2d instead of Gs)"""
    S, E, R = w.S, list(w.E), len(w.E)
    ns = w.problem["equation"] == "navier_stokes"
    segs = {}
    for kind in ("elements", "interfaces", "mortars", "boundaries"):
        seg = perk.list(kind)[1]
        segs[kind] = [int(seg[R - 1 - r + 1] - seg[R - 1 - r]) for r in range(R)]   # per member r
    halo = perk.halo_counts() if ns else None

    def active(r, i):
        return i == 1 or i >= S - E[r] + 2

    def lazy(r, i):
        return 2 <= i <= S - E[r] + 2

    def tr(r, i):
        return 256 if lazy(r, i) else 128

    fused = ns and br1_fused()
    out = {"volume_stage": 0, "surface": 0}
    if ns:
        out.update(br1_gradients=0)
        if not fused:
            out.update(br1_gradient_traces=0)
    for i in range(1, S + 1):
        for r in range(R):
            if not active(r, i):
                continue
            ne, ni, nm, nb = (segs[k][r] for k in ("elements", "interfaces", "mortars", "boundaries"))
            rl = max(r - 1, 0)                     # member of a mortar's large side
            if i == 1:
                vb = 1536
            elif i < S:
                vb = 2048 if lazy(r, i) else 2560
            else:
                vb = 2048
            out["volume_stage"] += ne * (vb + (384 if ns else 0))
            out["surface"] += ni * (2 * tr(r, i) + 2 * 128 + (2 * 96 if ns else 0))
            out["surface"] += nm * (tr(rl, i) + 2 * tr(r, i) + 3 * 128 + (3 * 96 if ns else 0))
            out["surface"] += nb * (tr(r, i) + 128)
            if ns:
                if fused:   # own state, the face neighbours' traces, Vt and Dv writes
                    out["br1_gradients"] += ne * ((1024 if lazy(r, i) else 512) + 2 * 384) + ni * 2 * tr(r, i) + \
                        nm * 2 * tr(rl, i) + (nm * 2 * tr(r, i) if active(rl, i) else 0)
                else:
                    out["br1_gradient_traces"] += ni * (2 * tr(r, i) + 2 * 96) + nm * (tr(rl, i) + 2 * tr(r, i) + 3 * 96)
                    out["br1_gradients"] += ne * ((1024 if lazy(r, i) else 512) + 3 * 384)   # + the Dv write
        if ns and fused:   # halo elements: lazy state, 4 lazy neighbour traces, Vt
            out["br1_gradients"] += int(halo["elements"][i - 1]) * (1024 + 4 * 256 + 384)
        elif ns:
            out["br1_gradient_traces"] += int(halo["interfaces"][i - 1]) * (2 * 256 + 2 * 96) + \
                int(halo["mortars"][i - 1]) * (3 * 256 + 3 * 96)
            out["br1_gradients"] += int(halo["elements"][i - 1]) * (1024 + 2 * 384)
    return out


def br1_fused():
    """the library forms the BR1 central traces inside k_grad2d (no k_gsurf2d launches, perk_build_flags)"""
    try:
        from paper_2403_05144_b200 import perk as _P
        return _P.build_flags()["br1_fused"]
    except Exception:
        return False


def _lib_sha():
    import hashlib
    try:
        with open(LIB, "rb") as f:
            return hashlib.sha256(f.read()).hexdigest()[:16]
    except OSError:
        return None


def kernel_counts(cfg):
    """ncu counts of the current kernels (profiles/r02_kernel_counts_cfg<cfg>.json, written by
    tools/kernel_counts.py from one ncu pass over every launch of one P-ERK step): per kernel kind the
    executed fp64 flops (2 DFMA + DMUL + DADD) and the cold-cache DRAM bytes per step."""
    path = os.path.join(ROOT, "profiles", f"r02_kernel_counts_cfg{cfg}.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    d["_path"] = os.path.relpath(path, ROOT)
    from paper_2403_05144_b200.build import source_sha16
    d["_current_build"] = d.get("src_sha16") == source_sha16() or d.get("lib_sha16") == _lib_sha()
    return d


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


def kernel_report(perk, w, cfg, timer, torch, elem_rhs_per_step, fp64, hbm):
    """Per kernel kind: flushed graph-replay time per step (perk_time_kernels_ex), algorithmic bytes
    (kernel_bytes_per_step) and executed fp64 flops (committed ncu counts) -> HBM and fp64 roofline
    fractions; the dominant kernel's larger fraction is the line's `roofline`."""
    fp64_peak, fp64_src = fp64
    hbm_peak, hbm_src = hbm
    ns = w.problem["equation"] == "navier_stokes"
    kinds = [0, 1] + (([5] if br1_fused() else [4, 5]) if ns else [])
    U0 = perk.initial_state(w.ic)
    ms_k = {k: perk.time_kernels(U0.clone(), w.dt, [k], reps=10, flush=timer.flush) for k in kinds}
    ms_all = perk.time_kernels(U0.clone(), w.dt, kinds, reps=10, flush=timer.flush)
    nbytes = kernel_bytes_per_step(perk, w)
    counts = kernel_counts(cfg)
    S = w.S
    roofs = {}
    for k in kinds:
        name = KIND_NAMES[k]
        ms = ms_k[k]
        cnt = (counts or {}).get("kinds", {}).get(name)
        gbs = nbytes[name] / (ms * 1e-3) / 1e9
        kname = KERNEL_OF_KIND[k] + ("<MODE_STAGE, NS>" if ns else "<MODE_STAGE>")
        traffic = round(cnt["dram_bytes_per_step"] / S) if cnt else None
        r_h = {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
               "frac": round(gbs / hbm_peak, 4), "traffic": traffic, "kernel": kname, "peak_source": hbm_src,
               "algorithmic_bytes_per_launch": round(nbytes[name] / S), "launches_per_step": S,
               "kernel_ms_per_launch": round(ms / S, 5), "kernel_ms_per_step": round(ms, 5)}
        r = {"hbm": r_h}
        if cnt and cnt.get("fp64_flops_per_step"):
            tf = cnt["fp64_flops_per_step"] / (ms * 1e-3) / 1e12
            r["alu"] = {"bound": "alu", "achieved": round(tf, 3), "peak": round(fp64_peak, 2), "unit": "TFLOP/s",
                        "frac": round(tf / fp64_peak, 4), "traffic": traffic, "kernel": kname,
                        "peak_source": fp64_src,
                        "fp64_flops_per_element_rhs": round(cnt["fp64_flops_per_step"] / elem_rhs_per_step, 1)}
        roofs[name] = r
    if counts:
        note = (f"traffic and flops: {counts['_path']} (ncu, one step, cold cache: ncu flushes caches between "
                f"replays); captured on {'this' if counts['_current_build'] else 'an EARLIER'} build of the library")
    else:
        note = "no ncu counts for this config: traffic null, no fp64 roofline"
    dom = max(kinds, key=lambda k: ms_k[k])
    rd = roofs[KIND_NAMES[dom]]
    best = max(rd.values(), key=lambda r: r["frac"])
    other = [r for r in rd.values() if r is not best]
    kern = {KIND_NAMES[k]: round(ms_k[k], 5) for k in kinds}
    kern["all_kinds_graph"] = round(ms_all, 5)
    kern["timing"] = "graph replays holding only that kind's launches of a step, L2 flushed between replays"
    return kern, roofs, best, (other[0] if other else None), note


def e2e_report(perk, w, U0, args, ws, elem_rhs_per_step, torch):
    """end to end through the public API with HOST buffers (pinned): perk_run_host copies the step's
    input state to the device, runs the step and copies the result back, inside the timed region"""
    n = perk.n_cells
    npe = 4 ** w.problem["dim"]
    Uh = U0[:n].cpu().pin_memory()
    e2e_steps = max(3, min(args.steps, 10))
    perk.run_host(Uh, w.dt, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        perk.run_host(Uh, w.dt, 1)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    h2d = int(n * w.nv * npe * 8)
    return {"value": round(ws * elem_rhs_per_step / e2e_s, 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": h2d, "ms_per_step": round(1e3 * e2e_s, 4),
            "how": "perk_run_host (pinned host state in, step, state out, synchronise), wall clock per call"}


def run_decomposed(args, torch, dist, ws, rank, local, dev):
    """N > 1: ONE problem decomposed over the N GPUs: each rank owns an E-weighted
    contiguous Morton range of the BASELINE mesh (DistributedPerk: the library's stage launches and
    pack / unpack kernels, the ghost blocks moved by NCCL point-to-point per stage).  Total work is
    fixed as N grows ("scaling": "strong"); value = the whole mesh's element-RHS per step / the
    slowest rank's device time per step."""
    from paper_2403_05144_b200 import DistributedPerk
    w = W.make(args.config)
    timer = _Timer(torch, dev, ws, dist)
    with ClockSampler(local) as clk:
        dp = DistributedPerk(w.problem, w.level_map, w.S, w.E, dist)
        U = dp.initial_state(w.ic)
        ts = timer.steps(lambda k: dp.step(U, w.dt), args.steps, args.warmup)
    ms = _max_over_ranks(torch, dist, ws, dev, float(np.mean(ts)))
    ev, st = dp.counters()
    t = torch.tensor([ev], dtype=torch.int64, device=dev)
    dist.all_reduce(t)
    elem_rhs_per_step = float(t.item()) / max(st, 1)
    f, c = dp.owned()
    if rank == 0:
        n = dp.p.n_cells
        npe = 4 ** w.problem["dim"]
        value = elem_rhs_per_step / (ms * 1e-3)
        line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator workloads/, DESIGN.md §3)",
                "config": {"workload": w.name, "cells": n, "nodes": n * npe, "S": w.S, "E": w.E,
                           "element_rhs_per_step": elem_rhs_per_step, "dt": w.dt,
                           "l2": "flushed between timed steps (256 MB write, outside the events)",
                           "parallelism": f"domain decomposition x{ws} (E-weighted Morton ranges, NCCL ghost "
                                          f"exchange per stage)", "rank0_owned_cells": c},
                "dof_stage_updates_per_s": round(value * npe, 1),
                "gpu_launches": (dp.p.launches_per_step() + w.S * len(dp.peers) * 2 * (2 if dp.ns else 1)) * args.steps,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    dp.close()
    dist.destroy_process_group()
    return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl")
    if ws > 1 and not args.replicas:
        try:
            return run_decomposed(args, torch, dist, ws, rank, local, torch.device("cuda", local))
        except Exception as ex:   # report it on the line and measure replicas instead of printing nothing
            args.decomposition_error = repr(ex)[:300]
            dist.barrier()
    dev = torch.device("cuda", local)
    timer = _Timer(torch, dev, ws, dist)
    fp64 = _fp64_peak()
    peaks, src = _peaks()
    hbm = (float(peaks.get("hbm_gbs", 6650.0)), src)

    from paper_2403_05144_b200 import Perk  # noqa: F401  (fails loudly without the CUDA library)
    with ClockSampler(local) as clk:
        w0 = W.make(args.config)
        # clock soak: untimed steps of the headline workload under load (>= 0.5 s)
        from paper_2403_05144_b200 import Perk as _P
        soak = _P(w0.problem, w0.level_map, w0.S, w0.E)
        Usoak = soak.initial_state(w0.ic)
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 0.5:
            for _ in range(10):
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
    kern = roofs = best = other = note = None
    if w.problem["dim"] == 2:
        kern, roofs, best, other, note = kernel_report(perk, w, args.config, timer, torch, elem_rhs_per_step, fp64, hbm)
    U0 = perk.initial_state(w.ic)
    e2e = e2e_report(perk, w, U0, args, ws, elem_rhs_per_step, torch)
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
                Ko = max(5, min(args.steps, 20))
                p2, _U, _w, r2 = measure_config(c, Ko, args.warmup, timer, torch, dist, ws, dev, order=order, amr=amr,
                                                 pattern=pattern, sc=sc)
                r2["dof_stage_updates_per_s"] = round(r2["value"] * 4 ** _w.problem["dim"], 1)
                r2["gpu_launches_per_step"] = p2.launches_per_step()
                if order == 2 and not amr and not pattern and not sc and _w.problem["dim"] == 2 and not _w.remesh_every:
                    # a static 2D configuration: the full per-kernel report, like the headline's
                    k2, ro2, b2, o2, n2 = kernel_report(p2, _w, c, timer, torch, r2["element_rhs_per_step"], fp64, hbm)
                    r2.update(kernel_ms_per_step=k2, roofline=b2, roofline_other=o2, roofline_kernels=ro2,
                              roofline_note=n2,
                              e2e=e2e_report(p2, _w, p2.initial_state(_w.ic), args, ws, r2["element_rhs_per_step"],
                                             torch))
                p2.close()
                others[f"cfg{item}"] = r2
            except Exception as ex:       # report, do not hide: the line records the failure
                others[f"cfg{item}"] = {"error": repr(ex)[:200]}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, budget_s=args.cpu_budget)

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
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": clocks,
        }
        if best:
            line["roofline"] = best
            line["roofline_other"] = other
            line["roofline_kernels"] = roofs
            line["roofline_note"] = note
        if others:
            line["other_configs"] = others
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if getattr(args, "decomposition_error", None):
            line["config"]["parallelism"] = f"replicas x{ws} (the domain decomposition failed: {args.decomposition_error})"
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _cells_per_member(m, R):
    mem = m.leaves()["member"]
    return [int((mem == r).sum()) for r in range(R)]


def oracle_sample(cfg, budget_s, threads):
    """The oracle as it stands on a bounded sample of BASELINE config `cfg`: whole P-ERK steps of the
    full mesh (restricted mode) while they fit the budget; if one step would not, the stage RHS
    evaluations of one P-ERK step in stage order (each F restricted to the members active at that
    stage, as in the step; the stage combinations, a few axpys, are left out), until the budget is
    spent.  Runs in this process; `threads` only labels the result (the caller sets ORACLE_OMP /
    OMP_NUM_THREADS)."""
    from oracle import oracle as O
    from oracle import tableau as T
    w = W.make(cfg)
    fam = T.family(w.S, w.E, w.alpha_rule)
    m = O.OracleMesh(w.problem, w.level_map, fam)
    U = m.initial_state(w.ic)
    R = len(w.E)
    cpm = _cells_per_member(m, R)
    t0 = time.perf_counter()
    m.rhs(U, (1 << R) - 1, 1)           # one full F: sizes the sample
    t_full = time.perf_counter() - t0
    ev_step = sum(e * c for e, c in zip(w.E, cpm))
    est_step = t_full * ev_step / m.n
    if est_step <= budget_s / 2:
        k = max(1, int(budget_s / max(est_step, 1e-9)))
        t1 = time.perf_counter()
        ev = m.step(U, w.dt, k)
        dt = time.perf_counter() - t1
        sample = f"{k} full P-ERK step(s) of {w.name} ({m.n} cells), restricted mode"
    else:
        ev, dt, nst = 0, 0.0, 0
        for i in range(1, w.S + 1):
            mask = sum(1 << r for r in range(R) if i == 1 or i >= w.S - w.E[r] + 2)
            t1 = time.perf_counter()
            m.rhs(U, mask, 1)
            dt += time.perf_counter() - t1
            ev += sum(c for r, c in enumerate(cpm) if (mask >> r) & 1)
            nst += 1
            if dt >= budget_s:
                break
        sample = (f"stage RHS evaluations 1..{nst} of one P-ERK step of {w.name} ({m.n} cells; each F restricted "
                  f"to the stage's active members, stage combinations omitted)")
    return {"value": round(ev / dt, 1), "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
            "seconds": round(dt, 2), "element_rhs": int(ev)}


def _oracle_subprocess(cfg, budget_s, threads):
    env = dict(os.environ, OMP_NUM_THREADS=str(threads), OMP_PROC_BIND="spread", OMP_PLACES="cores")
    env.pop("ORACLE_OMP", None)
    if threads > 1:
        env["ORACLE_OMP"] = "1"
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-worker", f"{cfg},{budget_s},{threads}"],
                         capture_output=True, text=True, env=env, timeout=30 * budget_s + 600)
    if out.returncode != 0:
        return {"error": out.stderr[-300:]}
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_baseline(cfg, budget_s=20.0):
    """The oracle (plain C) on this host: all cores (OpenMP build, bitwise the serial results) and one
    thread, each on a bounded sample of the same workload (oracle_sample); `value` / `cores` are the
    all-core run's."""
    nproc = os.cpu_count() or 1
    allc = _oracle_subprocess(cfg, budget_s, nproc)
    one = _oracle_subprocess(cfg, budget_s, 1)
    res = dict(allc) if "value" in allc else {"value": None, "unit": UNIT, "cores": nproc, "kind": "oracle",
                                               "sample": None, "error": allc.get("error")}
    res["cpu_model"] = _cpu_model()
    res["nproc"] = nproc
    res["single_thread"] = one
    return res


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


def reference_steps(cfg, K, Wm, cap_s):
    """--impl reference worker: the oracle (OpenMP build on all cores when ORACLE_OMP=1) runs Wm
    warm-up and then up to K whole P-ERK steps of the full mesh, stopping early once cap_s seconds
    of timed steps are spent (a bounded sample)."""
    from oracle import oracle as O
    from oracle import tableau as T
    w = W.make(cfg)
    fam = T.family(w.S, w.E, w.alpha_rule)
    m = O.OracleMesh(w.problem, w.level_map, fam)
    U = m.initial_state(w.ic)
    ev = 0
    for _ in range(Wm):
        ev = m.step(U, w.dt, 1)
    tot, dt, k = 0, 0.0, 0
    while k < K and dt < cap_s:
        t1 = time.perf_counter()
        tot += m.step(U, w.dt, 1)
        dt += time.perf_counter() - t1
        k += 1
    return {"value": round(tot / dt, 1), "steps": k, "seconds": round(dt, 2), "ms_per_step": round(1e3 * dt / k, 3),
            "cells": m.n, "element_rhs_per_step": int(ev), "workload": w.name}


def run_reference(args):
    """The reference arm (tier framing): the oracle as it stands, on the box's host cores (OpenMP build,
    all cores), whole P-ERK steps of the same workload; rank 0 only."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    nproc = os.cpu_count() or 1
    env = dict(os.environ, ORACLE_OMP="1", OMP_NUM_THREADS=str(nproc), OMP_PROC_BIND="spread", OMP_PLACES="cores")
    cap = 150.0
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--reference-worker",
                          f"{args.config},{args.steps},{args.warmup},{cap}"], capture_output=True, text=True, env=env)
    if out.returncode != 0:
        print(json.dumps({"impl": "reference", "unavailable": "oracle run failed: " + out.stderr[-200:]}), flush=True)
        return
    r = json.loads(out.stdout.strip().splitlines()[-1])
    sample = (f"{r['steps']} full P-ERK step(s) of {r['workload']} ({r['cells']} cells), restricted mode, "
              f"{nproc} OpenMP threads (requested --steps {args.steps}; stops after ~{cap:.0f} s of timed steps)")
    line = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": ws, "steps": r["steps"],
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator workloads/)",
            "config": {"workload": r["workload"], "cells": r["cells"], "element_rhs_per_step": r["element_rhs_per_step"]},
            "impl": "reference",
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": nproc, "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--extra", default="3,1,2,4,4i,3p3,3alt,3early,3sc,5sc",
                    help="other BASELINE configs measured into other_configs (comma list, 'Np3' = config N "
                         "with the P-ERK3 family, 'Ni' = config N with indicator-driven AMR, "
                         "'Nalt' / 'Nearly' = config N with the alternating / early-shared stage pattern, or 'none')")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent replicas of the workload instead of one decomposed problem")
    ap.add_argument("--profile-only", action="store_true",
                    help="build the workload and run warmup+steps P-ERK steps only (short ncu target)")
    ap.add_argument("--oracle-worker", default=None, help=argparse.SUPPRESS)      # cfg,budget_s,threads
    ap.add_argument("--reference-worker", default=None, help=argparse.SUPPRESS)   # cfg,K,W,cap_s
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.oracle_worker:
        c, b, t = args.oracle_worker.split(",")
        print(json.dumps(oracle_sample(int(c), float(b), int(t))), flush=True)
    elif args.reference_worker:
        c, k, wm, cap = args.reference_worker.split(",")
        print(json.dumps(reference_steps(int(c), int(k), int(wm), float(cap))), flush=True)
    elif args.profile_only:
        run_profile_only(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
