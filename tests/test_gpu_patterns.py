"""GPU parity of the stage-pattern variants and alternative weights: alternating,
early-shared and explicit non-nested evaluated-stage sets (P:l.642-700), Heun / Ralston weights
(P:l.439-442), on 2D Euler (multi-launch path), 1D (single-CTA step and multi-launch path) and
across device re-meshes; states <= 1e-10 per conserved variable, element-RHS counters exact, lists
bit-exact, per-stage launch sizes = the member-sorted prefix down to the lowest evaluating member."""
from fractions import Fraction as Fr

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from oracle import tableau as T
from gpu_util import TOL, gpu_state_numpy, rel_err_per_var

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

NON_NESTED_16 = [[1, 5, 9, 16], [1, 2, 4, 6, 8, 10, 12, 16], "standard"]


def _pair(w, pattern, c_S=Fr(1, 2), problem=None, level_map=None, max_cells=None):
    from paper_2403_05144_b200 import Perk
    problem = problem or w.problem
    lm = w.level_map if level_map is None else level_map
    fam = T.family(w.S, w.E, w.alpha_rule, pattern=pattern, c_S=c_S)
    ora = O.OracleMesh(problem, lm, fam)
    gpu = Perk(problem, lm, w.S, w.E, max_cells=max_cells or problem["max_cells"], pattern=pattern,
               c_S=float(c_S))
    return fam, ora, gpu


def _check_counts(fam, gpu):
    """stage-i launch size = the items the stage needs: elements / interfaces / boundaries of evaluating
    members, mortars with an evaluating fine or coarse side (nested patterns: the member-sorted prefix;
    non-nested: the per-stage lists)"""
    lv = gpu.leaves()
    mem_el = lv["member"]
    members = {"elements": (mem_el, None), "interfaces": (gpu.faces("interfaces")[1], None),
               "boundaries": (gpu.faces("boundaries")[1], None)}
    rec, mfine = gpu.faces("mortars")
    members["mortars"] = (mfine, mem_el[rec[:, 0]] if len(rec) else np.zeros(0, np.int32))
    for kind, (m1, m2) in members.items():
        ca = gpu.count_active(kind)
        for i in range(1, fam["S"] + 1):
            on = np.array([i in fam["stages"][r] for r in range(fam["R"])])
            need = on[m1] if m2 is None else (on[m1] | on[m2])
            assert ca[i - 1] == int(need.sum()), (kind, i, ca[i - 1], int(need.sum()))


def _run(w, fam, ora, gpu, steps):
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    ev_o = ora.step(Uo, w.dt, steps)
    gpu.step(Ug, w.dt, steps)
    torch.cuda.synchronize()
    gpu.sync()
    ev_g, st_g = gpu.counters()
    assert st_g == steps and ev_g == ev_o
    return Uo, gpu_state_numpy(gpu, Ug)


@pytest.mark.parametrize("pattern", ["alternating", "early", NON_NESTED_16], ids=str)
@pytest.mark.parametrize("c_S", [Fr(1, 2), Fr(1), Fr(2, 3)], ids=str)
def test_euler2d_patterns(pattern, c_S):
    w = W.make(3, n_base=16)
    fam, ora, gpu = _pair(w, pattern, c_S)
    lo, lg = ora.leaves(), gpu.leaves()
    assert all(np.array_equal(lo[k], lg[k]) for k in ("fx", "fy", "level", "member"))
    _check_counts(fam, gpu)
    Uo, Ug = _run(w, fam, ora, gpu, 20)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_euler2d_alternating_full_size():
    w = W.make(3)
    fam, ora, gpu = _pair(w, "alternating")
    Uo, Ug = _run(w, fam, ora, gpu, 1)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


@pytest.mark.parametrize("pattern", ["alternating", NON_NESTED_16], ids=str)
def test_remesh_with_patterns(pattern):
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 8, 16]
    fam, ora, gpu = _pair(w, pattern, max_cells=4 * W.configs.count_leaves(w))
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    for k in range(1, 4):
        ora.step(Uo, w.dt, 5)
        gpu.step(Ug, w.dt, 5)
        lm = w.level_map_seq(k)
        new = O.OracleMesh(w.problem, lm, fam)
        Uo = O.transfer(ora, new, Uo)
        ora = new
        gpu.repartition(lm, Ug)
        gpu.sync()
        _check_counts(fam, gpu)
    ora.step(Uo, w.dt, 5)
    gpu.step(Ug, w.dt, 5)
    torch.cuda.synchronize()
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL


@pytest.mark.parametrize("cfg,kw", [(1, {}), (2, {}), (2, {"n_base": 2048})], ids=["cfg1", "cfg2", "cfg2_big"])
@pytest.mark.parametrize("pattern", ["alternating", "early"])
def test_1d_patterns(cfg, kw, pattern):
    """cfg 1/2 run the single-CTA step kernel; n_base 2048 the two-launch-per-stage path"""
    w = W.make(cfg, **kw)
    fam, ora, gpu = _pair(w, pattern)
    Uo, Ug = _run(w, fam, ora, gpu, 30)
    assert rel_err_per_var(Ug, Uo).max() <= TOL
    if kw:
        assert gpu.launches_per_step() > 1


def test_heun_standard_1d_and_2d():
    for w in (W.make(2), W.make(3, n_base=16)):
        fam, ora, gpu = _pair(w, "standard", Fr(1))
        Uo, Ug = _run(w, fam, ora, gpu, 10)
        assert rel_err_per_var(Ug, Uo).max() <= TOL


@pytest.mark.parametrize("pattern", ["alternating", "early", [[1, 11, 21, 32], [1, 3, 5, 7, 9, 11, 13, 32],
                                                              "standard", "standard"]], ids=str)
def test_navier_stokes_patterns(pattern):
    """Navier-Stokes (BR1) with non-standard stage patterns: the superset member prefix per stage
    with its halo; surplus members see their lazy stage state"""
    w = W.make(5, n_base=8)
    fam, ora, gpu = _pair(w, pattern)
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    ora.step(Uo, w.dt, 10)
    gpu.step(Ug, w.dt, 10)
    torch.cuda.synchronize()
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL
    R = len(w.E)
    for mask in (1, (1 << R) - 1, 0b0101):
        dUo = ora.rhs(Uo, mask)
        dUg = gpu_state_numpy(gpu, gpu.rhs(Ug, mask))
        torch.cuda.synchronize()
        scale = np.abs(ora.rhs(Uo)).max(axis=(0, 2))
        assert (np.abs(dUg - dUo).max(axis=(0, 2)) / scale).max() <= TOL


def test_bad_masks_rejected():
    from paper_2403_05144_b200.perk import PerkError, tableau_p2
    w3 = W.make(3, n_base=8)
    with pytest.raises(PerkError):
        tableau_p2(w3.S, w3.E, pattern=[[1, 2, 16], [1, 2, 4, 5, 6, 7, 8, 16], "standard"])


def test_maximum_stage_count_s64():
    """S = PERK_MAX_STAGES = 64 (stage masks use all 64 bits), standard and alternating"""
    w = W.make(3, n_base=8)
    w.S, w.E = 64, [16, 32, 64]
    dt = w.dt * 4
    for pattern in ("standard", "alternating"):
        fam, ora, gpu = _pair(w, pattern)
        Uo = ora.initial_state(w.ic)
        Ug = gpu.initial_state(w.ic)
        ev_o = ora.step(Uo, dt, 2)
        gpu.step(Ug, dt, 2)
        torch.cuda.synchronize()
        gpu.sync()
        assert gpu.counters()[0] == ev_o
        assert gpu.launches_per_step() == 2 * 64
        assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL


def test_non_nested_superset_path(monkeypatch):
    """the 2D superset-prefix path (used when per-stage lists would exceed their memory budget):
    forced with PERK_STAGE_LISTS=0; surplus members' faces computed, their elements skipped"""
    monkeypatch.setenv("PERK_STAGE_LISTS", "0")
    w = W.make(3, n_base=16)
    fam, ora, gpu = _pair(w, NON_NESTED_16)
    # launch sizes are the member-sorted prefixes down to the lowest evaluating member
    _, seg = gpu.list("elements")
    ca = gpu.count_active("elements")
    for i in range(1, fam["S"] + 1):
        rmin = min(r for r in range(fam["R"]) if i in fam["stages"][r])
        assert ca[i - 1] == seg[fam["R"] - rmin]
    Uo, Ug = _run(w, fam, ora, gpu, 20)
    assert rel_err_per_var(Ug, Uo).max() <= TOL
