"""GPU parity: the CUDA path (libperk_b200.so through its C ABI) against the oracle on identical
seeded inputs.  Index lists bit-exact; states <= 1e-10 max relative error per conserved variable
(BASELINE.json north_star).  Sizes: every BASELINE config's full mesh (lists, one RHS, a few steps
at full size), full step counts where the oracle finishes in seconds, plus small ragged meshes,
boundaries, re-meshing and degenerate cases."""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from oracle import tableau as T
from gpu_util import TOL, build_pair, compare_mesh, expected_face_table, gpu_state_numpy, rel_err_per_var

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _run_both(w, steps, ora, gpu, mode=1):
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    assert np.abs(gpu_state_numpy(gpu, Ug) - Uo).max() < 1e-13 * max(1.0, np.abs(Uo).max())
    ora.step(Uo, w.dt, steps, mode=mode)
    gpu.step(Ug, w.dt, steps)
    torch.cuda.synchronize()
    gpu.sync()
    return Uo, gpu_state_numpy(gpu, Ug)


# ----------------------------------------------------------------------------------------------
# lists (a1-a3): bit-exact
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_lists_full_size(cfg):
    w = W.make(cfg)
    ora, gpu = build_pair(w)
    assert ora.n == gpu.n_cells
    compare_mesh(ora, gpu)


@pytest.mark.parametrize("seed", range(8))
def test_lists_random_small_2d(seed):
    rng = np.random.default_rng(100 + seed)
    nb, L = int(rng.choice([3, 4, 5, 8])), int(rng.integers(1, 4))
    T_ = (rng.integers(0, L + 1, size=(nb << L, nb << L)) * (rng.random((nb << L, nb << L)) < 0.1)).astype(np.int32)
    lm = W.balance(T_, L, (True, True))
    w = W.make(3, n_base=nb)
    p = W.configs._problem(2, "euler", "fluxdiff", "hll", nb, L, 0.0, 10.0)
    R = min(L + 1, 3)
    w.S, w.E = 16, [4, 8, 16][3 - R:]
    ora, gpu = build_pair(w, problem=p, level_map=lm)
    compare_mesh(ora, gpu)


def test_lists_nonperiodic_boundaries():
    w = W.make(3, n_base=8)
    p = dict(w.problem, periodic=(0, 1), bc_state=(1.0, 0.1, 0.0, 2.5))
    ora, gpu = build_pair(w, problem=p)
    assert ora.face_counts()["boundaries"] > 0
    compare_mesh(ora, gpu)


def test_unbalanced_rejected():
    from paper_2403_05144_b200 import PerkError
    lm = np.zeros((8, 8), np.uint8)
    lm[0:2, 0:2] = 2
    lm = W.leafify(lm, 2).astype(np.uint8)
    p = W.configs._problem(2, "euler", "fluxdiff", "hll", 2, 2, 0.0, 1.0)
    from paper_2403_05144_b200 import Perk
    with pytest.raises(PerkError) as ei:
        Perk(p, lm, 16, [4, 8, 16])
    assert ei.value.code == -2


def test_capacity_rejected():
    from paper_2403_05144_b200 import Perk, PerkError
    w = W.make(3, n_base=8)
    with pytest.raises(PerkError) as ei:
        Perk(w.problem, w.level_map, w.S, w.E, max_cells=10)
    assert ei.value.code == -3


# ----------------------------------------------------------------------------------------------
# one RHS per partition mask (a5-a10 without the stage combination)
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_rhs_eval_masks_full_size(cfg):
    w = W.make(cfg)
    ora, gpu = build_pair(w)
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    R = len(w.E)
    for mask in sorted({(1 << R) - 1, 1, 1 << (R - 1), (1 << R) - 2}):
        dUo = ora.rhs(Uo, mask, mode=0)       # the definition: full F, then the mask I^(r)
        dUg = gpu_state_numpy(gpu, gpu.rhs(Ug, mask))
        # a single RHS is a difference of O((2/h) |f|) terms: rounding-order differences scale with
        # (2/h_min) max|U|, not with |dU| (the 1e-10 state criterion applies to the full runs below)
        scale = 2.0 / w.problem["h_min"] * np.abs(Uo).max()   # magnitude of the summed flux terms
        for v in range(dUo.shape[1]):
            tol = 1e-12 * np.abs(dUo[:, v]).max() + 4e-14 * scale
            assert np.abs(dUg[:, v] - dUo[:, v]).max() <= tol, (mask, v)
        # unmasked partitions are exactly zero
        mem = ora.leaves()["member"]
        off = ~np.isin(mem, [r for r in range(R) if (mask >> r) & 1])
        assert np.all(dUg[off] == 0.0)


# ----------------------------------------------------------------------------------------------
# full runs: the P-ERK step (a5-a13)
# ----------------------------------------------------------------------------------------------
def test_cfg1_full_run():
    w = W.make(1)
    ora, gpu = build_pair(w)
    Uo, Ug = _run_both(w, w.steps, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL
    ev, st = gpu.counters()
    assert st == w.steps and ev == 320 * w.steps


def test_cfg2_full_run():
    w = W.make(2)
    ora, gpu = build_pair(w)
    Uo, Ug = _run_both(w, w.steps, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL
    ev, st = gpu.counters()
    assert ev == 2560 * w.steps


def test_cfg3_small_full_steps():
    """cfg-3 structure on a 16^2 base (several tiles + ragged tails), the full 500 steps."""
    w = W.make(3, n_base=16)
    ora, gpu = build_pair(w)
    assert ora.face_counts()["mortars"] > 0
    Uo, Ug = _run_both(w, w.steps, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_cfg3_full_size_steps():
    """BASELINE cfg 3 mesh (62,932 cells) in the bench launch configuration, 2 steps."""
    w = W.make(3)
    ora, gpu = build_pair(w)
    Uo, Ug = _run_both(w, 2, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL
    ev, st = gpu.counters()
    assert ev == 2 * 713596


def test_cfg4_initial_mesh_steps():
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 6, 10, 16]
    ora, gpu = build_pair(w)
    Uo, Ug = _run_both(w, 20, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_boundary_variant_2d():
    """weakly imposed Dirichlet faces (a8) on a non-periodic x direction."""
    w = W.make(3, n_base=8)
    p = dict(w.problem, periodic=(0, 1), bc_state=(1.0, 1.0, 1.0, 1.0 / 0.4 + 1.0))
    ora, gpu = build_pair(w, problem=p)
    Uo, Ug = _run_both(w, 30, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_boundary_variant_1d():
    w = W.make(2, n_base=64, w1=16, w2=4, steps=200)
    p = dict(w.problem, periodic=(0, 1), bc_state=(1.0, 1.0, 1.0 / 0.4 + 0.5))
    ora, gpu = build_pair(w, problem=p)
    assert ora.face_counts()["boundaries"] == 2
    Uo, Ug = _run_both(w, w.steps, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_single_level_reduction():
    """uniform mesh at the finest level: GPU multirate == oracle single-rate S-stage P-ERK."""
    w = W.make(3, n_base=8, steps=10)
    lm = np.full_like(w.level_map, w.problem["max_level"])
    from paper_2403_05144_b200 import Perk
    ora = O.OracleMesh(w.problem, lm, T.family(16, [16], "taylor"))
    gpu = Perk(w.problem, lm, 16, [4, 8, 16])
    Uo, Ug = _run_both(w, w.steps, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_cfg1_coarse_only_mesh():
    """degenerate: no cell at the finest level (all cells in the lowest member)."""
    w = W.make(1)
    lm = np.zeros_like(w.level_map)
    ora, gpu = build_pair(w, level_map=lm)
    compare_mesh(ora, gpu)
    Uo, Ug = _run_both(w, 50, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_e2e_host_buffers_match_device_path():
    w = W.make(3, n_base=16)
    from paper_2403_05144_b200 import Perk
    gpu = Perk(w.problem, w.level_map, w.S, w.E)
    U = gpu.initial_state(w.ic)
    n = gpu.n_cells
    Uh = U[:n].cpu().pin_memory()
    gpu.step(U, w.dt, 3)
    gpu.run_host(Uh, w.dt, 3)
    torch.cuda.synchronize()
    assert torch.equal(Uh, U[:n].cpu())


# ----------------------------------------------------------------------------------------------
# dynamic re-mesh (a1-a4 on the device)
# ----------------------------------------------------------------------------------------------
def test_repartition_lists_and_transfer():
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 6, 10, 16]
    fam = T.family(w.S, w.E, "taylor")
    ora, gpu = build_pair(w, max_cells=4 * W.configs.count_leaves(w))
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    for k in range(1, 5):
        ora.step(Uo, w.dt, 5)
        gpu.step(Ug, w.dt, 5)
        lm = w.level_map_seq(k)
        ora_new = O.OracleMesh(w.problem, lm, fam)
        Uo = O.transfer(ora, ora_new, Uo)
        ora = ora_new
        gpu.repartition(lm, Ug)
        gpu.sync()
        compare_mesh(ora, gpu)
        assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL
    ora.step(Uo, w.dt, 5)
    gpu.step(Ug, w.dt, 5)
    torch.cuda.synchronize()
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL


# ----------------------------------------------------------------------------------------------
# Navier-Stokes, BR1 (a10): cfg 5 structure
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("n_base", [8, 256])
def test_ns_rhs_eval_masks(n_base):
    """one RHS per upward-closed mask and the full mask; 256 = the BASELINE cfg-5 mesh (305,827 cells)"""
    w = W.make(5, n_base=n_base)
    ora, gpu = build_pair(w)
    assert ora.face_counts()["mortars"] > 0
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    R = len(w.E)
    masks = [(1 << R) - 1, 1 << (R - 1), ((1 << R) - 1) & ~1]
    for mask in masks:
        dUo = ora.rhs(Uo, mask, mode=0)
        dUg = gpu_state_numpy(gpu, gpu.rhs(Ug, mask))
        scale = 2.0 / w.problem["h_min"] * np.abs(Uo).max()
        for v in range(4):
            tol = 1e-12 * np.abs(dUo[:, v]).max() + 4e-14 * scale
            assert np.abs(dUg[:, v] - dUo[:, v]).max() <= tol, (mask, v)


@pytest.mark.parametrize("n_base", [8, 256])
def test_ns_face_table(n_base):
    """the fused BR1 pass's device-built face-neighbour table (an index structure: bit-exact) against
    the table written out from the oracle's face records; 256 = the BASELINE cfg-5 mesh"""
    from paper_2403_05144_b200 import perk as P
    w = W.make(5, n_base=n_base)
    ora, gpu = build_pair(w)
    if not P.build_flags()["br1_fused"]:
        pytest.skip("library built without BR1_FUSED")
    assert np.array_equal(gpu.face_table(), expected_face_table(ora))


def test_face_table_unsupported_for_euler():
    w = W.make(3, n_base=8)
    ora, gpu = build_pair(w)
    with pytest.raises(Exception) as ei:
        gpu.face_table()
    assert ei.value.code == -6


def test_cfg5_small_full_run():
    """cfg-5 structure (4 levels, {4, 8, 16, 32}, BR1) on an 8^2 base, the full 200 steps"""
    w = W.make(5, n_base=8)
    ora, gpu = build_pair(w)
    Uo, Ug = _run_both(w, w.steps, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL
    ev, st = gpu.counters()
    cnt = ora.count_active("elements")
    assert st == w.steps and ev == int(cnt.sum()) * w.steps


def test_cfg5_medium_steps():
    w = W.make(5, n_base=32)
    ora, gpu = build_pair(w)
    Uo, Ug = _run_both(w, 5, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_cfg5_full_size_step():
    """BASELINE cfg 5 mesh (305,827 cells) in the bench launch configuration, 1 step (~50 s oracle)"""
    w = W.make(5)
    ora, gpu = build_pair(w)
    Uo, Ug = _run_both(w, 1, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_ns_single_level_reduction():
    w = W.make(5, n_base=8, steps=10)
    lm = np.full_like(w.level_map, w.problem["max_level"])
    from paper_2403_05144_b200 import Perk
    ora = O.OracleMesh(w.problem, lm, T.family(32, [32], "taylor"))
    gpu = Perk(w.problem, lm, 32, [4, 8, 16, 32])
    Uo, Ug = _run_both(w, w.steps, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_ns_free_stream_gpu():
    w = W.make(5, n_base=8)
    from paper_2403_05144_b200 import Perk
    gpu = Perk(w.problem, w.level_map, w.S, w.E)
    U = gpu.initial_state(lambda x, y: np.stack([1.2 + 0 * x, 0.36 + 0 * x, -0.6 + 0 * x, 60.0 + 0 * x]))
    dU = gpu_state_numpy(gpu, gpu.rhs(U))
    assert np.abs(dU).max() <= 1e-13 * (2.0 / w.problem["h_min"]) * 60.0


def test_ns_nonperiodic_rejected():
    from paper_2403_05144_b200 import Perk, PerkError
    w = W.make(5, n_base=8)
    p = dict(w.problem, periodic=(0, 1))
    with pytest.raises(PerkError) as ei:
        Perk(p, w.level_map, w.S, w.E)
    assert ei.value.code == -6


def test_cfg4_full_size_remesh():
    """BASELINE cfg 4 (64^2 base, Lmax 4, {4,6,10,16,28}, ~77.7k cells) in the bench launch
    configuration: 5 steps, one device re-mesh (lists bit-exact, transfer), 5 more steps."""
    w = W.make(4)
    fam = T.family(w.S, w.E, w.alpha_rule)
    ora, gpu = build_pair(w)
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    ora.step(Uo, w.dt, 5)
    gpu.step(Ug, w.dt, 5)
    lm = w.level_map_seq(1)
    ora_new = O.OracleMesh(w.problem, lm, fam)
    Uo = O.transfer(ora, ora_new, Uo)
    ora = ora_new
    gpu.repartition(lm, Ug)
    gpu.sync()
    compare_mesh(ora, gpu)
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL
    ora.step(Uo, w.dt, 5)
    gpu.step(Ug, w.dt, 5)
    torch.cuda.synchronize()
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL


def test_cfg4_long_run_many_remeshes():
    """cfg-4 structure on a 16^2 base (Lmax 3): 100 steps with a device re-mesh every 5 steps (20
    re-meshes), the cadence of BASELINE cfg 4."""
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 6, 10, 16]
    fam = T.family(w.S, w.E, "taylor")
    ora, gpu = build_pair(w, max_cells=4 * W.configs.count_leaves(w))
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    for k in range(1, 21):
        ora.step(Uo, w.dt, 5)
        gpu.step(Ug, w.dt, 5)
        lm = w.level_map_seq(k)
        ora_new = O.OracleMesh(w.problem, lm, fam)
        Uo = O.transfer(ora, ora_new, Uo)
        ora = ora_new
        gpu.repartition(lm, Ug)
    gpu.sync()
    compare_mesh(ora, gpu)
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL


# ----------------------------------------------------------------------------------------------
# P-ERK3 families: explicit tableaux from workloads/perk3.py, general weights b
# ----------------------------------------------------------------------------------------------
def _pair_p3(w, fam, problem=None, level_map=None):
    from paper_2403_05144_b200 import Perk
    problem = problem or w.problem
    lm = w.level_map if level_map is None else level_map
    ora = O.OracleMesh(problem, lm, fam)
    gpu = Perk(problem, lm, fam["S"], fam["E"], family=fam, max_cells=problem["max_cells"])
    return ora, gpu


def test_p3_cfg3_small_100_steps():
    from workloads import perk3 as P3
    w = W.make(3, n_base=16)
    ora, gpu = _pair_p3(w, P3.family3(16, (4, 8, 16)))
    Uo, Ug = _run_both(w, 100, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_p3_cfg3_full_size_steps():
    from workloads import perk3 as P3
    w = W.make(3)
    ora, gpu = _pair_p3(w, P3.family3(16, (4, 8, 16)))
    Uo, Ug = _run_both(w, 2, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_p3_1d_euler_full_run():
    from workloads import perk3 as P3
    w = W.make(2)
    ora, gpu = _pair_p3(w, P3.family3(12, (3, 6, 12)))
    Uo, Ug = _run_both(w, w.steps, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_p3_ns_small_run():
    from workloads import perk3 as P3
    w = W.make(5, n_base=8)
    ora, gpu = _pair_p3(w, P3.family3(32, (4, 8, 16, 32)))
    Uo, Ug = _run_both(w, 50, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_p3_rejects_E2_member():
    from paper_2403_05144_b200 import Perk, PerkError
    from workloads import perk3 as P3
    w = W.make(3, n_base=8)
    fam = dict(P3.family3(16, (4, 8, 16)))
    fam["E"] = [2, 8, 16]
    with pytest.raises(PerkError) as ei:
        Perk(w.problem, w.level_map, 16, fam["E"], family=fam)
    assert ei.value.code == -1


@pytest.mark.parametrize("order", [2, 3])
def test_ns_repartition(order):
    """BR1 Navier-Stokes across device re-meshes (cfg-4 structure, KH state, mu = 1e-3), P-ERK2 and
    P-ERK3: lists bit-exact after each re-mesh, states <= 1e-10."""
    from paper_2403_05144_b200 import Perk
    from workloads import perk3 as P3
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 6, 10, 16]
    prob = dict(w.problem, equation="navier_stokes", mu=1e-3, prandtl=0.72)
    fam = T.family(w.S, w.E, "taylor") if order == 2 else P3.family3(w.S, w.E)
    cap = 4 * W.configs.count_leaves(w)
    ora = O.OracleMesh(prob, w.level_map, fam)
    gpu = Perk(prob, w.level_map, w.S, w.E, max_cells=cap, family=None if order == 2 else fam)
    Uo = ora.initial_state(w.ic)
    Ug = gpu.initial_state(w.ic)
    for k in range(1, 4):
        ora.step(Uo, w.dt, 5)
        gpu.step(Ug, w.dt, 5)
        lm = w.level_map_seq(k)
        ora_new = O.OracleMesh(prob, lm, fam)
        Uo = O.transfer(ora, ora_new, Uo)
        ora = ora_new
        gpu.repartition(lm, Ug)
        gpu.sync()
        compare_mesh(ora, gpu)
        from paper_2403_05144_b200 import perk as P
        if P.build_flags()["br1_fused"]:
            assert np.array_equal(gpu.face_table(), expected_face_table(ora))
    ora.step(Uo, w.dt, 5)
    gpu.step(Ug, w.dt, 5)
    torch.cuda.synchronize()
    assert rel_err_per_var(gpu_state_numpy(gpu, Ug), Uo).max() <= TOL


@pytest.mark.parametrize("cfg", [2, 3])
def test_e2_member(cfg):
    """degenerate member E = 2 (evaluates stages 1 and S only; its stage-S state is the lazy
    U_n + dt c_S K_1 while U_n is updated in place at stage S): 1D single-CTA path and 2D path"""
    w = W.make(cfg, n_base=64 if cfg == 2 else 16, **({"w1": 16, "w2": 4} if cfg == 2 else {}))
    w.S, w.E = 8, [2, 4, 8]
    ora, gpu = build_pair(w)
    Uo, Ug = _run_both(w, 40, ora, gpu)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


def test_repartition_errors_latch():
    """capacity overflow and an unbalanced map during a device re-mesh are reported by the next
    synchronising call (no host round trip inside perk_repartition)"""
    from paper_2403_05144_b200 import Perk, PerkError
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 6, 10, 16]
    n0 = W.configs.count_leaves(w)
    gpu = Perk(w.problem, w.level_map, w.S, w.E, max_cells=n0)
    U = gpu.initial_state(w.ic)
    fine = np.minimum(w.level_map + 1, 3).astype(np.uint8)   # every leaf refined once: ~4x the cells
    gpu.repartition(fine, U)
    with pytest.raises(PerkError) as ei:
        gpu.sync()
    assert ei.value.code == -3
    gpu2 = Perk(w.problem, w.level_map, w.S, w.E, max_cells=4 * n0)
    U2 = gpu2.initial_state(w.ic)
    bad = np.zeros_like(w.level_map)
    bad[0:8, 0:8] = 3                                         # a level-3 block next to level 0
    gpu2.repartition(bad, U2)
    with pytest.raises(PerkError) as ei:
        gpu2.sync()
    assert ei.value.code == -2


def test_capacity_large_overflow_is_clean():
    """a large overflow (cap = n/4 on the ~78k-cell cfg-4 mesh, at perk_init and during a
    device re-mesh) must latch PERK_ECAPACITY without an out-of-bounds access: no sticky CUDA error,
    so a fresh context on the same device still runs and matches the oracle."""
    from paper_2403_05144_b200 import Perk, PerkError
    w = W.make(4)
    n0 = W.configs.count_leaves(w)
    with pytest.raises(PerkError) as ei:
        Perk(w.problem, w.level_map, w.S, w.E, max_cells=n0 // 4)
    assert ei.value.code == -3
    coarse = W.make(4, widths=(0.3, 0.15, 0.06, 0.0))       # no level-4 band: fewer cells
    nc = W.configs.count_leaves(coarse)
    assert nc < n0
    gpu = Perk(w.problem, coarse.level_map, w.S, w.E, max_cells=nc)
    U = gpu.initial_state(w.ic)
    gpu.repartition(w.level_map, U)                          # needs n0 > cap cells
    with pytest.raises(PerkError) as ei:
        gpu.sync()
    assert ei.value.code == -3
    torch.cuda.synchronize()                                 # raises on a sticky device error
    small = W.make(3, n_base=16, steps=3)
    ora, g2 = build_pair(small)
    Uo, Ug = _run_both(small, small.steps, ora, g2)
    assert max(rel_err_per_var(Ug, Uo)) < TOL


def test_1d_repartition_unsupported():
    from paper_2403_05144_b200 import Perk, PerkError
    w = W.make(1)
    gpu = Perk(w.problem, w.level_map, w.S, w.E)
    U = gpu.initial_state(w.ic)
    with pytest.raises(PerkError) as ei:
        gpu.repartition(w.level_map, U)
    assert ei.value.code == -6


def test_capacity_large_overflow_ns_is_clean():
    """the same for a Navier-Stokes context, whose re-mesh also builds the fused BR1 face table from the
    (overflowed) face records: a latched PERK_ECAPACITY, no sticky device error"""
    from paper_2403_05144_b200 import Perk, PerkError
    w = W.make(5, n_base=64)
    n0 = W.configs.count_leaves(w)
    with pytest.raises(PerkError) as ei:
        Perk(w.problem, w.level_map, w.S, w.E, max_cells=n0 // 4)
    assert ei.value.code == -3
    torch.cuda.synchronize()
    small = W.make(5, n_base=8, steps=2)
    ora, g2 = build_pair(small)
    Uo, Ug = _run_both(small, small.steps, ora, g2)
    assert rel_err_per_var(Ug, Uo).max() <= TOL


@pytest.mark.parametrize("cfg,sc", [(3, False), (5, False), (5, True), (3, True)])
def test_launches_per_step_matches_profile(cfg, sc):
    """perk_launches_per_step (bench.py's gpu_launches) equals the kernels one eager profiled step launches"""
    from paper_2403_05144_b200 import Perk
    w = W.make(cfg, n_base=8)
    prob = dict(w.problem, shock_capturing=W.configs.SHOCK_CAPTURING) if sc else w.problem
    gpu = Perk(prob, w.level_map, w.S, w.E)
    U = gpu.initial_state(w.ic)
    _, nl = gpu.profile_step(U, w.dt)
    assert sum(nl) == gpu.launches_per_step()
