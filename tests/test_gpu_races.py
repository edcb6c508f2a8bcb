"""Race checks of the staged kernels without compute-sanitizer (its racecheck is closed on this GPU
pool): results must not depend on the schedule.

* persistent grids capped to 1, 3 and 37 CTAs (PERK_VOL_BLOCKS / PERK_GRAD_BLOCKS / PERK_SURF_BLOCKS):
  every element group then runs through few CTAs' cp.async staging rings, back to back -- the
  state after several P-ERK steps must be bitwise that of the default grid (Euler, Navier-Stokes,
  shock capturing with the atomicMax smoothing);
* the debug library (libperk_debug.so) with perk_debug_jitter: every thread of k_vol2d / k_grad2d
  sleeps a pseudo-random 0..4 us at each warp barrier and asynchronous-copy wait, so the threads of a
  warp drift apart; a missing __syncwarp or cp.async wait would read stale shared memory.  Jittered
  == unjittered, bitwise.
* the alternating sweep direction of consecutive stage kernels (StageParams::rev, DESIGN §5 item 4) is a
  schedule change only: PERK_SWEEP=0 (every launch forward) must give the same bits.
Each case runs in a subprocess (the grid caps are read at perk_init; the debug library is loaded
instead of the release one there)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import workloads as W
from paper_2403_05144_b200 import Perk, perk
case, jitter = sys.argv[1], int(sys.argv[2])
cfg, nb = {{"euler": (3, 16), "ns": (5, 32), "sc": (3, 16)}}[case]
w = W.make(cfg, n_base=nb)
if case == "sc":
    w.problem = dict(w.problem, shock_capturing=W.configs.SHOCK_CAPTURING)
    w.ic = W.configs.contact_band(w.ic)
if jitter:
    assert perk.lib().perk_debug_jitter(jitter) == 0
p = Perk(w.problem, w.level_map, w.S, w.E)
U = p.initial_state(w.ic)
p.step(U, w.dt, 4)
torch.cuda.synchronize()
p.sync()
a = U[: p.n_cells].cpu().numpy()
print(json.dumps({{"sha": hashlib.sha256(a.tobytes()).hexdigest(), "finite": bool(np.isfinite(a).all())}}))
"""


def _run(case, env_extra, jitter=0):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), case, str(jitter)], capture_output=True,
                         text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("case", ["euler", "ns", "sc"])
def test_grid_size_independent(case):
    ref = _run(case, {})
    assert ref["finite"]
    for nb in ("1", "3", "37"):
        r = _run(case, {"PERK_VOL_BLOCKS": nb, "PERK_GRAD_BLOCKS": nb, "PERK_SURF_BLOCKS": nb})
        assert r["sha"] == ref["sha"], (case, nb)


@pytest.mark.parametrize("case", ["euler", "ns"])
def test_jitter_debug_build(case):
    dbg = os.path.join(ROOT, "paper_2403_05144_b200", "lib", "libperk_debug.so")
    if not os.path.exists(dbg):
        from paper_2403_05144_b200 import build
        build.build_debug(force=False)
    env = {"PERK_LIB_PATH": dbg}
    ref = _run(case, env, 0)
    for seed in (1, 12345):
        r = _run(case, env, seed)
        assert r["sha"] == ref["sha"], (case, seed)
    # the debug build computes the same numbers as the release build
    assert _run(case, {})["sha"] == ref["sha"]


@pytest.mark.parametrize("case", ["euler", "ns", "sc"])
def test_sweep_direction_independent(case):
    """Every stage kernel walks its lists opposite to its predecessor (L2 reuse); items are independent,
    so the all-forward schedule gives bitwise the same state."""
    assert _run(case, {"PERK_SWEEP": "0"})["sha"] == _run(case, {})["sha"]
