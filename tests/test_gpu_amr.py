"""GPU parity of the indicator-driven AMR path: perk_amr_indicator /
perk_amr_adapt (amr.cuh) against the oracle (perk_oracle.c section 8) on identical seeded states.

* indicators per leaf: Hennemann-Gassner (all five variables), Loehner, enstrophy, within 1e-10
  (the floating-point order of the modal sums / derivatives differs);
* the adapted level map bit-exact: equal to the oracle controller's map on the GPU's indicator
  values, and equal to the oracle's own map unless a leaf's two indicator values straddle a
  threshold, which is only allowed within 1e-9 (relative) of it;
* full cfg-4 size, periodic and non-periodic meshes, Navier-Stokes, and a 10-cycle
  step / adapt / repartition loop compared with the oracle mesh-by-mesh and state-by-state;
* launch count, error codes.
"""
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

HG = dict(indicator="hennemann_gassner", variable="rho", base_level=0, med_level=2, max_level=4,
          med_threshold=0.01, max_threshold=0.1, alpha_max=0.5, alpha_min=0.001)
LOHNER = dict(indicator="lohner", variable="v_x", base_level=0, med_level=2, max_level=4,
              med_threshold=0.003, max_threshold=0.03, f_wave=0.2)


def _perturbed(gpu, ora, w, amp, seed=7):
    """the cfg-4 state plus seeded per-node noise (so that every indicator spans its range);
    returns (oracle array, device tensor) holding identical values"""
    Uo = ora.initial_state(w.ic)
    rng = np.random.default_rng(seed)
    scale = amp * rng.random((ora.n, 1, 1)) ** 3            # a few elements strongly perturbed
    Uo = Uo * (1.0 + scale * rng.standard_normal(Uo.shape))
    Ug = gpu.alloc_state()
    Ug[: ora.n] = torch.from_numpy(Uo).cuda()
    return np.ascontiguousarray(Uo), Ug


def _thresholds(amr):
    return np.array([amr["med_threshold"], amr["max_threshold"]])


def _compare_maps(ora, lm_o, lm_g, ind_o, ind_g, amr):
    """The GPU map must be EXACTLY the oracle controller's map on the GPU's own indicator values
    (controller + balance bit-exact given the same inputs), and every leaf whose decision differs
    between the two indicators (a value on the other side of a threshold) must be a near-tie
    (within 1e-9 relative of that threshold; the indicators themselves agree to <= 1e-10).  With no
    such leaf this is lm_g == lm_o.  Returns the number of tie leaves."""
    ind_g = np.asarray(ind_g, np.float64)
    assert ind_g.shape == ind_o.shape
    lm_from_g = ora.amr_adapt(None, amr, indicator=ind_g)
    assert np.array_equal(lm_from_g, lm_g), "GPU controller / balance differs from the oracle's on the same indicator"
    th = _thresholds(amr)
    side_o = ind_o[:, None] <= th[None, :]
    side_g = ind_g[:, None] <= th[None, :]
    ties = np.nonzero((side_o != side_g).any(axis=1))[0]
    if len(ties) == 0:
        assert np.array_equal(lm_o, lm_g)
        return 0
    tol = 1e-9 * max(np.abs(th).max(), 1e-300)
    for e in ties:
        k = np.nonzero(side_o[e] != side_g[e])[0]
        assert (np.abs(ind_o[e] - th[k]) <= tol).all(), (e, ind_o[e], ind_g[e], th[k])
    return len(ties)


@pytest.mark.parametrize("amr", [
    dict(HG, variable="rho"), dict(HG, variable="p"), dict(HG, variable="rho_p"), dict(HG, variable="v_x"),
    dict(HG, variable="v_y"), LOHNER, dict(LOHNER, variable="rho_p"), "enstrophy"], ids=str)
def test_indicator_parity(amr):
    w = W.make(4, n_base=16)
    amr = w.meta["amr"] if amr == "enstrophy" else amr
    ora, gpu = build_pair(w)
    Uo, Ug = _perturbed(gpu, ora, w, 0.05)
    io = ora.amr_indicator(Uo, amr)
    ig = gpu.amr_indicator(Ug, amr).cpu().numpy()
    scale = max(np.abs(io).max(), 1e-300)
    assert np.abs(ig - io).max() <= 1e-10 * scale, (np.abs(ig - io).max(), scale)
    assert io.max() > io.min()                                      # a non-trivial field


@pytest.mark.parametrize("amr", [HG, LOHNER, "enstrophy"], ids=str)
@pytest.mark.parametrize("n_base,L,amp", [(16, 4, 0.02), (64, 4, 0.01), (12, 1, 0.02), (12, 2, 0.02),
                                          (6, 6, 0.02)])
def test_adapt_map_parity(amr, n_base, L, amp):
    """maximum levels 1..6 (one balance CTA holds 1..256 base cells), ragged base grids"""
    w = W.make(4, n_base=n_base, max_level=L, widths=(0.3, 0.15, 0.06, 0.015, 0.008, 0.004)[:L])
    amr = w.meta["amr"] if amr == "enstrophy" else dict(amr, max_level=min(4, L), med_level=min(2, L))
    ora, gpu = build_pair(w)
    Uo, Ug = _perturbed(gpu, ora, w, amp)
    lm_o = ora.amr_adapt(Uo, amr)
    lm_g = gpu.amr_adapt(Ug, amr).cpu().numpy()
    gpu.sync()
    _compare_maps(ora, lm_o, lm_g, ora.amr_indicator(Uo, amr), gpu.amr_indicator(Ug, amr).cpu().numpy(), amr)
    assert not np.array_equal(lm_o, w.level_map)                   # the controller changed the mesh


@pytest.mark.parametrize("periodic", [(0, 0), (1, 0)])
def test_adapt_nonperiodic(periodic):
    w = W.make(4, n_base=16)
    prob = dict(w.problem, periodic=periodic, bc_state=(1.0, 0.0, 0.0, 2.5))
    ora, gpu = build_pair(w, problem=prob)
    Uo, Ug = _perturbed(gpu, ora, w, 0.02)
    amr = dict(HG, max_level=4)
    lm_o = ora.amr_adapt(Uo, amr)
    lm_g = gpu.amr_adapt(Ug, amr).cpu().numpy()
    _compare_maps(ora, lm_o, lm_g, ora.amr_indicator(Uo, amr), gpu.amr_indicator(Ug, amr).cpu().numpy(), amr)


def test_adapt_navier_stokes():
    w = W.make(5, n_base=16)
    ora, gpu = build_pair(w)
    Uo, Ug = _perturbed(gpu, ora, w, 0.02)
    amr = dict(indicator="enstrophy", base_level=0, med_level=1, max_level=3, med_threshold=0.05,
               max_threshold=0.5)
    io = ora.amr_indicator(Uo, amr)
    lm_o = ora.amr_adapt(Uo, amr)
    lm_g = gpu.amr_adapt(Ug, amr).cpu().numpy()
    _compare_maps(ora, lm_o, lm_g, io, gpu.amr_indicator(Ug, amr).cpu().numpy(), amr)


def test_adapt_loop_state_and_lists():
    """10 cycles of 5 steps + adapt + repartition (the indicator-driven cfg 4 at n_base 16)"""
    w = W.make(4, n_base=16)
    amr = w.meta["amr"]
    fam = T.family(w.S, w.E, w.alpha_rule)
    ora, gpu = build_pair(w)
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    lm_g = torch.zeros(w.level_map.shape, dtype=torch.uint8, device="cuda")
    changed = 0
    for k in range(10):
        ora.step(Uo, w.dt, 5)
        gpu.step(Ug, w.dt, 5)
        lm_o = ora.amr_adapt(Uo, amr)
        ig = gpu.amr_indicator(Ug, amr).cpu().numpy()
        gpu.amr_adapt(Ug, amr, out=lm_g)
        gpu.repartition(lm_g, Ug)
        gpu.sync()
        assert _compare_maps(ora, lm_o, lm_g.cpu().numpy(), ora.amr_indicator(Uo, amr), ig, amr) == 0
        ora_new = O.OracleMesh(w.problem, lm_o, fam)
        changed += int(ora_new.n != ora.n)
        Uo = O.transfer(ora, ora_new, Uo)
        ora = ora_new
        compare_mesh(ora, gpu)
        assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL
    assert changed > 0


def test_launches_and_errors():
    w = W.make(4, n_base=16)
    ora, gpu = build_pair(w)
    assert gpu.amr_launches() == w.problem["max_level"] + 3
    U = gpu.initial_state(w.ic)
    from paper_2403_05144_b200.perk import PerkError
    for bad in (dict(HG, max_level=5), dict(HG, med_level=0, base_level=1), dict(HG, med_threshold=1.0),
                dict(HG, alpha_min=0.7), dict(LOHNER, f_wave=-1.0)):
        with pytest.raises(PerkError) as ei:
            gpu.amr_adapt(U, bad)
        assert ei.value.code == -1
    w1 = W.make(2)
    o1, g1 = build_pair(w1)
    with pytest.raises(PerkError) as ei:
        g1.amr_indicator(g1.initial_state(w1.ic), HG)
    assert ei.value.code == -6


def test_adapt_cycle_full_size():
    """BASELINE cfg 4 at full size (77,728 leaves): 2 steps, enstrophy adapt + device repartition,
    1 step; maps, lists and state against the oracle"""
    w = W.make(4)
    amr = w.meta["amr"]
    fam = T.family(w.S, w.E, w.alpha_rule)
    ora, gpu = build_pair(w)
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    ora.step(Uo, w.dt, 2)
    gpu.step(Ug, w.dt, 2)
    lm_o = ora.amr_adapt(Uo, amr)
    ig = gpu.amr_indicator(Ug, amr).cpu().numpy()
    lm_g = gpu.amr_adapt(Ug, amr)
    gpu.repartition(lm_g, Ug)
    gpu.sync()
    assert _compare_maps(ora, lm_o, lm_g.cpu().numpy(), ora.amr_indicator(Uo, amr), ig, amr) == 0
    new = O.OracleMesh(w.problem, lm_o, fam)
    Uo = O.transfer(ora, new, Uo)
    compare_mesh(new, gpu)
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL
    new.step(Uo, w.dt, 1)
    gpu.step(Ug, w.dt, 1)
    torch.cuda.synchronize()
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL


@pytest.mark.parametrize("variant", ["perk3", "alternating"])
def test_adapt_loop_with_perk3_and_patterns(variant):
    """indicator-driven re-meshing combined with the P-ERK3 family / a non-nested stage pattern"""
    from paper_2403_05144_b200 import Perk
    from workloads import perk3 as P3
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 8, 16]
    amr = dict(w.meta["amr"], max_level=3, med_level=2)
    if variant == "perk3":
        fam = P3.family3(w.S, w.E)
        gpu = Perk(w.problem, w.level_map, w.S, w.E, family=fam, max_cells=4 * W.configs.count_leaves(w))
    else:
        fam = T.family(w.S, w.E, w.alpha_rule, pattern="alternating")
        gpu = Perk(w.problem, w.level_map, w.S, w.E, pattern="alternating", max_cells=4 * W.configs.count_leaves(w))
    ora = O.OracleMesh(w.problem, w.level_map, fam)
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    for _ in range(3):
        ora.step(Uo, w.dt, 4)
        gpu.step(Ug, w.dt, 4)
        lm_o = ora.amr_adapt(Uo, amr)
        ig = gpu.amr_indicator(Ug, amr).cpu().numpy()
        lm_g = gpu.amr_adapt(Ug, amr)
        gpu.repartition(lm_g, Ug)
        gpu.sync()
        assert _compare_maps(ora, lm_o, lm_g.cpu().numpy(), ora.amr_indicator(Uo, amr), ig, amr) == 0
        new = O.OracleMesh(w.problem, lm_o, fam)
        Uo = O.transfer(ora, new, Uo)
        ora = new
        lo, lg = ora.leaves(), gpu.leaves()
        assert all(np.array_equal(lo[k], lg[k]) for k in ("fx", "fy", "level", "member"))
        assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL
    ora.step(Uo, w.dt, 4)
    gpu.step(Ug, w.dt, 4)
    torch.cuda.synchronize()
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL
