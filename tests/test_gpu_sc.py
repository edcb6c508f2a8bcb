"""GPU parity of the subcell shock capturing (sc.cuh + k_vol2d<., ., true>) against
the oracle (perk_oracle.c section 9, pinned by tests/test_oracle_sc.py) on identical seeded states.

* blending factors (raw and smoothed) per leaf, and rhs_eval for every partition mask, Euler and
  Navier-Stokes, HLL and Rusanov, indicator-driven and fixed alpha (0.5, 1), mortar meshes;
* P-ERK steps (stage-wise alpha on the lazy / buffered stage states, the halo across mortars)
  with a contact discontinuity that switches the blending on in a band of elements: cfg-3 and
  cfg-5 structures, a P-ERK3 family, the full cfg-3 mesh, and repartition cycles;
* launch counts, on / off switching (off again equals the unblended path bitwise), error codes.
"""
import os

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from oracle import tableau as T
from gpu_util import TOL, build_pair, compare_mesh, gpu_state_numpy, rel_err_per_var

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

SC = W.configs.SHOCK_CAPTURING


def _with_sc(w, sc=SC, surface=None):
    p = dict(w.problem)
    p["shock_capturing"] = sc
    if surface:
        p["surface"] = surface
    return p


def _jump_ic(ic):
    return W.configs.contact_band(ic)


def _pair(w, problem, max_cells=None):
    return build_pair(w, problem=problem, max_cells=max_cells)


def _to_dev(gpu, Uo):
    Ug = gpu.alloc_state()
    Ug[: Uo.shape[0]] = torch.from_numpy(np.ascontiguousarray(Uo)).cuda()
    return Ug


def _run_both(w, ora, gpu, steps, ic):
    Uo = ora.initial_state(ic)
    Ug = gpu.initial_state(ic)
    ora.step(Uo, w.dt, steps)
    gpu.step(Ug, w.dt, steps)
    torch.cuda.synchronize()
    return Uo, gpu_state_numpy(gpu, Ug)


@pytest.mark.parametrize("cfg,sc,surface", [
    (3, SC, None), (3, dict(SC, smooth=False), None), (3, dict(SC, alpha_fixed=1.0), None),
    (3, dict(SC, alpha_fixed=0.5), "rusanov"), (3, dict(SC, variable="rho", alpha_max=1.0), "rusanov"),
    (5, SC, None), (5, dict(SC, alpha_fixed=1.0), None)])
def test_alpha_and_rhs_eval_masks(cfg, sc, surface):
    w = W.make(cfg, n_base=16)
    ora, gpu = _pair(w, _with_sc(w, sc, surface))
    assert ora.face_counts()["mortars"] > 0
    ic = _jump_ic(w.ic)
    Uo = ora.initial_state(ic)
    Ug = _to_dev(gpu, Uo)
    ro, so = ora.sc_alpha(Uo)
    rg, sg = gpu.sc_alpha(Ug)
    rg, sg = rg.cpu().numpy(), sg.cpu().numpy()
    assert np.max(np.abs(rg - ro)) <= TOL and np.max(np.abs(sg - so)) <= TOL
    if sc.get("alpha_fixed") is None:
        assert 0 < np.count_nonzero(so) < ora.n          # blended and pure-DG elements
    # masked RHS errors are measured on the scale of the full F per variable: a masked subset can
    # have a RHS many orders below the terms that cancel in it (cfg 5, finest member only: max |d rho|
    # 7e-6 against max |F_rho| 463; a 1e-15 relative perturbation of U moves it by 1.6e-6 of its own
    # maximum in the oracle alone), A8
    R = len(w.E)
    Fo = ora.rhs(Uo)
    scale = np.abs(Fo).max(axis=(0, 2))
    for mask in sorted({(1 << R) - 1, 1, 1 << (R - 1), ((1 << R) - 1) ^ 1}):
        dUo = ora.rhs(Uo, mask)
        dUg = gpu_state_numpy(gpu, gpu.rhs(Ug, mask))
        torch.cuda.synchronize()
        err = np.abs(dUg - dUo).max(axis=(0, 2)) / scale
        assert err.max() <= TOL, (mask, err)


@pytest.mark.parametrize("epi", ["1", "0"])
def test_cfg3_structure_steps(epi):
    """epi 1 (default): the next stage's alpha of buffered elements from the k_vol2d epilogue;
    epi 0: every stage's alpha from k_sc_alpha"""
    w = W.make(3, n_base=16)
    os.environ["PERK_SC_EPI"] = epi
    try:
        ora, gpu = _pair(w, _with_sc(w))
    finally:
        del os.environ["PERK_SC_EPI"]
    Uo, Ug = _run_both(w, ora, gpu, 40, _jump_ic(w.ic))
    assert rel_err_per_var(Ug, Uo).max() <= TOL
    _, sm = ora.sc_alpha(Uo)
    assert 0 < np.count_nonzero(sm) < ora.n


@pytest.mark.parametrize("epi", ["default", "0"])
def test_cfg5_structure_steps(epi):
    w = W.make(5, n_base=16)
    if epi != "default":
        os.environ["PERK_SC_EPI"] = epi
    try:
        ora, gpu = _pair(w, _with_sc(w))
    finally:
        os.environ.pop("PERK_SC_EPI", None)
    Uo, Ug = _run_both(w, ora, gpu, 20, _jump_ic(w.ic))
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_perk3_family_steps():
    from workloads import perk3
    from paper_2403_05144_b200 import Perk
    w = W.make(3, n_base=16)
    fam3 = perk3.family3(16, (4, 8, 16))
    p = _with_sc(w)
    ora = O.OracleMesh(p, w.level_map, fam3)
    gpu = Perk(p, w.level_map, fam3["S"], fam3["E"], family=fam3, max_cells=p["max_cells"])
    Uo, Ug = _run_both(w, ora, gpu, 20, _jump_ic(w.ic))
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_full_cfg3_mesh_steps():
    """BASELINE cfg-3 mesh (62,932 cells), bench launch configuration, 2 steps"""
    w = W.make(3)
    ora, gpu = _pair(w, _with_sc(w))
    Uo, Ug = _run_both(w, ora, gpu, 2, _jump_ic(w.ic))
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_repartition_cycles():
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 6, 10, 16]
    fam = T.family(w.S, w.E, "taylor")
    p = _with_sc(w)
    ora, gpu = build_pair(w, problem=p, max_cells=4 * W.configs.count_leaves(w))
    ic = _jump_ic(w.ic)
    Uo = ora.initial_state(ic)
    Ug = gpu.initial_state(ic)
    for k in range(1, 4):
        ora.step(Uo, w.dt, 5)
        gpu.step(Ug, w.dt, 5)
        lm = w.level_map_seq(k)
        new = O.OracleMesh(p, lm, fam)
        Uo = O.transfer(ora, new, Uo)
        ora = new
        gpu.repartition(lm, Ug)
        gpu.sync()
        compare_mesh(ora, gpu)
        assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL
    ora.step(Uo, w.dt, 5)
    gpu.step(Ug, w.dt, 5)
    torch.cuda.synchronize()
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL


def test_switch_on_off_and_launch_counts():
    w = W.make(3, n_base=8)
    ora, gpu = build_pair(w)
    ic = _jump_ic(w.ic)
    U0 = gpu.initial_state(ic)
    base = gpu.launches_per_step()
    a = U0.clone()
    gpu.step(a, w.dt, 3)
    gpu.set_shock_capturing(SC)
    assert gpu.launches_per_step() == base + w.S      # blending factors; smoothing inside k_surf2d
    b = U0.clone()
    gpu.step(b, w.dt, 3)
    os.environ["PERK_SC_FUSED"] = "0"                 # stand-alone smoothing kernel
    try:
        gpu.set_shock_capturing(SC)
    finally:
        del os.environ["PERK_SC_FUSED"]
    assert gpu.launches_per_step() == base + 2 * w.S
    b2 = U0.clone()
    gpu.step(b2, w.dt, 3)
    gpu.set_shock_capturing(dict(SC, smooth=False))
    assert gpu.launches_per_step() == base + w.S
    torch.cuda.synchronize()
    assert torch.equal(b, b2)                 # atomicMax smoothing: order-independent, bitwise equal
    gpu.set_shock_capturing(None)
    assert gpu.launches_per_step() == base
    c = U0.clone()
    gpu.step(c, w.dt, 3)
    torch.cuda.synchronize()
    assert torch.equal(a, c)                 # off again: bitwise the unblended path
    assert not torch.equal(a, b)


def test_error_codes():
    from paper_2403_05144_b200 import Perk, PerkError
    w = W.make(3, n_base=8)
    gpu = Perk(w.problem, w.level_map, w.S, w.E)
    with pytest.raises(PerkError):
        gpu.set_shock_capturing(dict(SC, alpha_max=1.5))
    with pytest.raises(PerkError):
        gpu.set_shock_capturing(dict(SC, alpha_min=0.7))
    w1 = W.make(2, n_base=64, w1=16, w2=4, steps=10)
    g1 = Perk(w1.problem, w1.level_map, w1.S, w1.E)
    with pytest.raises(PerkError):
        g1.set_shock_capturing(SC)


@pytest.mark.parametrize("surface", ["hll", "rusanov"])
def test_nonperiodic_boundary_steps(surface):
    """weakly imposed Dirichlet faces on a non-periodic x direction (a8) with shock capturing: the
    boundary faces enter the subcell FV through the unchanged surface term, no smoothing across them"""
    w = W.make(3, n_base=8)
    p = dict(_with_sc(w, surface=surface), periodic=(0, 1), bc_state=(1.0, 1.0, 1.0, 1.0 / 0.4 + 1.0))
    ora, gpu = build_pair(w, problem=p)
    assert ora.face_counts()["boundaries"] > 0
    Uo, Ug = _run_both(w, ora, gpu, 30, _jump_ic(w.ic))
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_amr_adapt_with_shock_capturing():
    """device indicator-driven AMR (perk_amr_adapt, f3) cycles with shock capturing on"""
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 6, 10, 16]
    fam = T.family(w.S, w.E, "taylor")
    p = _with_sc(w)
    amr = dict(indicator="hennemann_gassner", variable="rho_p", base_level=0, med_level=1, max_level=3,
               med_threshold=0.01, max_threshold=0.1)
    ora, gpu = build_pair(w, problem=p)     # capacity: every finest cell a leaf
    ic = _jump_ic(w.ic)
    Uo = ora.initial_state(ic)
    Ug = gpu.initial_state(ic)
    for _ in range(3):
        ora.step(Uo, w.dt, 5)
        gpu.step(Ug, w.dt, 5)
        torch.cuda.synchronize()
        assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL
        lm_g = gpu.amr_adapt(Ug, amr)
        lm_o = ora.amr_adapt(Uo, amr)
        assert np.array_equal(lm_g.cpu().numpy(), lm_o)
        new = O.OracleMesh(p, lm_o, fam)
        Uo = O.transfer(ora, new, Uo)
        ora = new
        gpu.repartition(lm_g, Ug)
        gpu.sync()
        compare_mesh(ora, gpu)
    ora.step(Uo, w.dt, 5)
    gpu.step(Ug, w.dt, 5)
    torch.cuda.synchronize()
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL


@pytest.mark.parametrize("pattern,stage_lists", [("alternating", "1"), ("alternating", "0"), ("early", "1"),
                                                 ([[1, 5, 9, 16], [1, 2, 4, 6, 8, 10, 12, 16], "standard"], "1")])
def test_stage_patterns_steps(pattern, stage_lists):
    """non-standard stage patterns (f2) with shock capturing: alpha of every element at every stage
    (per-stage hot arrays, and the superset-prefix path with PERK_STAGE_LISTS=0)"""
    from paper_2403_05144_b200 import Perk
    w = W.make(3, n_base=16)
    p = _with_sc(w)
    fam = T.family(w.S, w.E, w.alpha_rule, pattern=pattern)
    ora = O.OracleMesh(p, w.level_map, fam)
    os.environ["PERK_STAGE_LISTS"] = stage_lists
    try:
        gpu = Perk(p, w.level_map, w.S, w.E, pattern=pattern)
    finally:
        del os.environ["PERK_STAGE_LISTS"]
    Uo, Ug = _run_both(w, ora, gpu, 20, _jump_ic(w.ic))
    assert rel_err_per_var(Ug, Uo).max() <= TOL
