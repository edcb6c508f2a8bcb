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


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            P = json.load(f)
        return P, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


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


def _volume_bytes_per_step(count_el, S, first):
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


FLOPS_PER_ELEMENT_RHS = None  # filled from DESIGN.md §5 model below


def flops_per_element_rhs():
    """Algorithmic fp64 flops of one 2D element RHS (DESIGN.md §5 count, FMA = 2 flops):
    48 two-point Ranocha fluxes x 96 + 16 nodes x 70 (primitives, 2 logs) + 64 x 6 (lift, Jacobian,
    epilogue)."""
    return 48 * 96 + 16 * 70 + 64 * 6


def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl")
    from paper_2403_05144_b200 import Perk

    w = W.make(args.config)
    dev = torch.device("cuda", local)
    perk = Perk(w.problem, w.level_map, w.S, w.E)
    U = perk.initial_state(w.ic)
    U0 = U.clone()
    n = perk.n_cells
    count_el = [int(x) for x in perk.count_active("elements")]
    elem_rhs_per_step = sum(count_el)
    npe = 4 ** w.problem["dim"]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def timed_steps(p, Ux, K, Wm):
        for _ in range(Wm):
            p.step(Ux, w.dt)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evs = []
        for _ in range(K):
            flush.fill_(1.0)                      # evict L2 between timed steps
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            p.step(Ux, w.dt)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    with ClockSampler(local) as clk:
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 0.5:          # clock soak: untimed steps under load
            for _ in range(50):
                perk.step(U, w.dt)
            torch.cuda.synchronize()
        times = timed_steps(perk, U, args.steps, args.warmup)
    ms = float(np.mean(times))
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ws * elem_rhs_per_step / (ms * 1e-3)

    # single-rate S-stage P-ERK on the same mesh and dt (multirate speedup, BASELINE north star)
    single = Perk(w.problem, w.level_map, w.S, [w.S])
    Us = single.initial_state(w.ic)
    ms_single = float(np.mean(timed_steps(single, Us, max(3, args.steps // 2), args.warmup)))
    single.close()

    # per-kernel device time of the same step: CUDA events around every launch on the launch stream
    prof_steps = 3
    ms_k = np.zeros(4)
    nl = np.zeros(4, dtype=np.int64)
    Up = U0.clone()
    for _ in range(prof_steps):
        m_, l_ = perk.profile_step(Up, w.dt)
        ms_k += np.array(m_)
        nl += np.array(l_)
    vol_ms_per_step = ms_k[1] / prof_steps
    surf_ms_per_step = ms_k[0] / prof_steps
    vol_bytes = _volume_bytes_per_step(count_el, w.S, None)
    peaks, src = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    achieved_gbs = vol_bytes / (vol_ms_per_step * 1e-3) / 1e9
    clk_max = float(peaks.get("sm_max_mhz", 1965.0))
    fp64_peak = 148 * 64 * 2 * clk_max * 1e6 / 1e12   # TFLOP/s: 148 SMs x 64 FP64 FMA/clk x 2
    achieved_tf = elem_rhs_per_step * flops_per_element_rhs() / (vol_ms_per_step * 1e-3) / 1e12
    roof_hbm = {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved_gbs / hbm, 4), "traffic": args.traffic,
                "kernel": "k_vol2d<MODE_STAGE> (volume + surface lift + Jacobian + stage epilogue)",
                "peak_source": src, "bytes_per_step": vol_bytes}
    roof_alu = {"bound": "alu", "achieved": round(achieved_tf, 3), "peak": round(fp64_peak, 2), "unit": "TFLOP/s",
                "frac": round(achieved_tf / fp64_peak, 4), "traffic": args.traffic,
                "kernel": roof_hbm["kernel"], "peak_source": "derived: 148 SM x 64 DFMA/clk x 2 x sm_max_mhz",
                "flops_per_element_rhs": flops_per_element_rhs()}
    roof = roof_alu if roof_alu["frac"] >= roof_hbm["frac"] else roof_hbm
    other = roof_hbm if roof is roof_alu else roof_alu

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

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, budget_s=args.cpu_budget)

    if rank == 0:
        launches = perk.launches_per_step()
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator workloads/, DESIGN.md §3)",
            "config": {"workload": w.name, "cells": n, "nodes": n * npe, "S": w.S, "E": w.E,
                       "element_rhs_per_step": elem_rhs_per_step, "dt": w.dt,
                       "l2": "flushed between timed steps (256 MB write, outside the events)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
            "dof_stage_updates_per_s": round(value * npe, 1),
            "scalar_dof_stage_updates_per_s": round(value * npe * w.nv, 1),
            "single_rate_ms_per_step": round(ms_single, 5),
            "multirate_speedup": round(ms_single / ms, 4),
            "ideal_multirate_speedup": round(w.S * n / elem_rhs_per_step, 4),
            "kernel_ms_per_step": {"surface": round(surf_ms_per_step, 5), "volume_stage": round(vol_ms_per_step, 5)},
            "roofline": roof, "roofline_other": other,
            "e2e": {"value": round(e2e_val, 1), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d},
            "gpu_launches": launches * args.steps,
            "clocks": clocks,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    perk.close()
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
    t0 = time.perf_counter()
    ev = m.step(U, w.dt, 1)                        # one warm-up step (no JIT; also sizes the sample)
    t_step = time.perf_counter() - t0
    K = max(1, min(args.steps, int(120.0 / max(t_step, 1e-9))))
    t1 = time.perf_counter()
    tot = m.step(U, w.dt, K)
    dt = time.perf_counter() - t1
    value = tot / dt
    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws, "steps": K,
            "warmup": 1, "ms_per_step": round(1e3 * dt / K, 3), "higher_is_better": True, "scaling": "weak",
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
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true",
                    help="build the workload and run warmup+steps P-ERK steps only (short ncu target)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per step of the dominant kernel from an ncu --set full capture")
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
