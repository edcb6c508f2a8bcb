"""Pins of the oracle's AMR indicators and level controller (perk_oracle.c section 8;
DESIGN.md A1-A6).  The paper names the indicators (Loehner on v_x, P:l.1440-1441; Hennemann-Gassner
on rho / rho*p, P:l.1548, l.1731, l.1886) and defines the enstrophy eps = 0.5 rho w.w with a
refinement threshold (P:l.1615-1622, eq. Enstrophy); the pins below are what the mathematics fixes:

* Hennemann-Gassner: nodal data built from single orthonormal Legendre tensor modes (numpy's
  Legendre series, not the oracle's Vandermonde) give the modal energy fractions in closed form,
  E = a^2 / (4 + a^2) etc., so a wrong normalisation, a wrong mode class (highest vs second
  highest, x vs y) or a transposed transform fails; E = 0 gives alpha = 1e-4 exactly (the
  logistic's definition); clipping by alpha_min / alpha_max; the five indicator variables;
* Loehner: hand-computed ratios (5/6, 5/8), zero on constants, invariance under positive scaling
  and under reflection of the element;
* enstrophy: exact vorticity of polynomial velocity fields (rigid rotation w = 2 Omega on every
  element size; cubic and quadratic fields w = 3 x^2 - 2 y);
* controller + balance: one level per adaptation, coarsening only with all four siblings, and the
  final map equal to the unique minimal 2:1-balanced refinement found by brute-force enumeration
  of all trees on tiny meshes (periodic and not), and equal to the workload generator's
  independent balance at larger sizes.
"""
import itertools

import numpy as np
import pytest
from numpy.polynomial import legendre as npleg

import workloads as W
from oracle import oracle as O
from oracle import tableau as T

G = 1.4
XI = np.array([-1.0, -1.0 / np.sqrt(5.0), 1.0 / np.sqrt(5.0), 1.0])
FAM = T.family(4, [4], "taylor")
S_HG = np.log((1 - 1e-4) / 1e-4)
T_HG = 0.5 * 10 ** (-1.8 * 4 ** 0.25)


def _prob(nb, L, periodic=(1, 1)):
    return W.configs._problem(2, "euler", "fluxdiff", "hll", nb, L, 0.0, 1.0, periodic=periodic)


def _mesh(nb=2, L=1, lm=None, periodic=(1, 1)):
    lm = np.zeros((nb << L, nb << L), np.uint8) if lm is None else lm
    return O.OracleMesh(_prob(nb, L, periodic), lm, FAM)


def _ptilde(k, x):
    c = np.zeros(k + 1)
    c[k] = 1.0
    return np.sqrt((2 * k + 1) / 2) * npleg.legval(x, c)


def _local_xy():
    """reference coordinates of node q = i + 4 j"""
    q = np.arange(16)
    return XI[q % 4], XI[q // 4]


def _state(m, rho, vx, vy, p):
    """conserved state from per-node primitive arrays of shape (16,) or (n, 16)"""
    shp = (m.n, 16)
    rho, vx, vy, p = (np.broadcast_to(np.asarray(a, np.float64), shp) for a in (rho, vx, vy, p))
    U = np.stack([rho, rho * vx, rho * vy, p / (G - 1) + 0.5 * rho * (vx * vx + vy * vy)], axis=1)
    return np.ascontiguousarray(U)


def _hg(ind_var="rho", alpha_max=1.0, alpha_min=0.0):
    return dict(indicator="hennemann_gassner", variable=ind_var, base_level=0, med_level=0, max_level=0,
                med_threshold=0.5, max_threshold=0.5, alpha_max=alpha_max, alpha_min=alpha_min)


def _alpha(E):
    return 1.0 / (1.0 + np.exp(-(S_HG / T_HG) * (E - T_HG)))


# ------------------------------------------------------------------------------------------
# A1 Hennemann-Gassner
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("modes,E_of", [
    ({(3, 0): 0.06}, lambda a: a[0] ** 2 / (4 + a[0] ** 2)),                    # highest mode in x
    ({(1, 3): 0.05}, lambda a: a[0] ** 2 / (4 + a[0] ** 2)),                    # highest mode in y
    ({(2, 1): 0.07}, lambda a: a[0] ** 2 / (4 + a[0] ** 2)),                    # second-highest class
    ({(2, 2): 0.08}, lambda a: a[0] ** 2 / (4 + a[0] ** 2)),
    ({(1, 1): 0.5}, lambda a: 0.0),                                             # resolved: E = 0
    ({(3, 0): 0.05, (2, 1): 0.2}, lambda a: max(a[0] ** 2 / (4 + a[0] ** 2 + a[1] ** 2),
                                                a[1] ** 2 / (4 + a[1] ** 2))),
    ({(0, 3): 0.2, (1, 2): 0.05}, lambda a: max(a[0] ** 2 / (4 + a[0] ** 2 + a[1] ** 2),
                                                a[1] ** 2 / (4 + a[1] ** 2))),
    # E near the threshold T (alpha ~ 0.2): "k <= N-1 AND l <= N-1" for the clipped sum matters
    ({(3, 0): 0.07, (2, 2): 0.03}, lambda a: max(a[0] ** 2 / (4 + a[0] ** 2 + a[1] ** 2),
                                                 a[1] ** 2 / (4 + a[1] ** 2))),
])
def test_hg_modal_energy_closed_form(modes, E_of):
    """field = 2 Pt_0(x) Pt_0(y) + sum a_kl Pt_k(x) Pt_l(y): sum of squares 4 + sum a_kl^2 (Parseval)"""
    m = _mesh()
    x, y = _local_xy()
    f = 2 * _ptilde(0, x) * _ptilde(0, y)
    for (k, l), a in modes.items():
        f = f + a * _ptilde(k, x) * _ptilde(l, y)
    want = _alpha(E_of(list(modes.values())))
    U = _state(m, f, 0.0, 0.0, 1.0)
    got = m.amr_indicator(U, _hg("rho"))
    assert np.allclose(got, want, rtol=1e-9, atol=1e-12), (got[0], want)


def test_hg_constant_is_1e4_and_clipping():
    m = _mesh()
    U = _state(m, 1.3, 0.2, -0.1, 0.9)
    assert np.allclose(m.amr_indicator(U, _hg("rho")), 1e-4, rtol=1e-9)          # exp(s) = (1 - 1e-4) / 1e-4
    assert np.all(m.amr_indicator(U, _hg("rho", alpha_min=0.001)) == 0.0)      # alpha < alpha_min -> 0
    x, y = _local_xy()
    U = _state(m, 2 * _ptilde(0, x) * _ptilde(0, y) + 0.9 * _ptilde(3, x) * _ptilde(0, y), 0, 0, 1)
    assert np.all(m.amr_indicator(U, _hg("rho", alpha_min=0.001)) == 1.0)      # alpha > 1 - alpha_min -> 1
    assert np.all(m.amr_indicator(U, _hg("rho", alpha_max=0.5, alpha_min=0.001)) == 0.5)


@pytest.mark.parametrize("var", ["rho", "p", "rho_p", "v_x", "v_y"])
def test_hg_indicator_variables(var):
    """the same modal field carried by each indicator variable (the others held so the variable is it)"""
    m = _mesh()
    x, y = _local_xy()
    a = 0.07
    f = 2 * _ptilde(0, x) * _ptilde(0, y) + a * _ptilde(3, x) * _ptilde(1, y)
    one, zero = np.ones(16), np.zeros(16)
    prim = {"rho": (f, zero, zero, one), "p": (one, zero, zero, f), "rho_p": (f, zero, zero, one),
            "v_x": (2 * one, f, 0.1 * one, one), "v_y": (2 * one, 0.1 * one, f, one)}[var]
    U = _state(m, *prim)
    got = m.amr_indicator(U, _hg(var))
    assert np.allclose(got, _alpha(a * a / (4 + a * a)), rtol=1e-9)


# ------------------------------------------------------------------------------------------
# A2 Loehner
# ------------------------------------------------------------------------------------------
def _lohner(var="v_x", f_wave=0.2):
    return dict(indicator="lohner", variable=var, base_level=0, med_level=0, max_level=0,
                med_threshold=0.5, max_threshold=0.5, f_wave=f_wave)


@pytest.mark.parametrize("row,want", [((0, 1, 0, 0), 5 / 6), ((1, 2, 1, 1), 5 / 8)])
def test_lohner_hand_values(row, want):
    """every x line carries `row` (v_x), so y lines are constant:
    (0,1,0,0): node 1: 2 / (2 + 0.2 * 2) = 5/6, node 2: 1 / (1 + 0.2) = 5/6;
    (1,2,1,1): node 1: 2 / (2 + 0.2 * 6) = 5/8, node 2: 1 / (1 + 0.2 * 5) = 1/2"""
    m = _mesh()
    vx = np.tile(np.array(row, np.float64), 4)
    U = _state(m, 2.0, vx, 0.0, 1.0)
    assert np.allclose(m.amr_indicator(U, _lohner()), want, rtol=1e-14)
    # the same data along y through v_y
    vy = np.repeat(np.array(row, np.float64), 4)
    U = _state(m, 2.0, 0.0, vy, 1.0)
    assert np.allclose(m.amr_indicator(U, _lohner("v_y")), want, rtol=1e-14)


def test_lohner_invariances():
    m = _mesh()
    rng = np.random.default_rng(3)
    f = 1 + 0.3 * rng.random((m.n, 16))
    base = m.amr_indicator(_state(m, f, 0, 0, 1), _lohner("rho"))
    assert np.all(base > 0)
    assert np.allclose(m.amr_indicator(_state(m, 7.5 * f, 0, 0, 1), _lohner("rho")), base, rtol=1e-13)
    flip = f.reshape(m.n, 4, 4)[:, ::-1, ::-1].reshape(m.n, 16)               # reflect x and y
    assert np.allclose(m.amr_indicator(_state(m, flip, 0, 0, 1), _lohner("rho")), base, rtol=1e-13)
    trans = f.reshape(m.n, 4, 4).transpose(0, 2, 1).reshape(m.n, 16)           # swap x and y
    assert np.allclose(m.amr_indicator(_state(m, trans, 0, 0, 1), _lohner("rho")), base, rtol=1e-13)
    assert np.all(m.amr_indicator(_state(m, 1.7, 0, 0, 1), _lohner("rho")) == 0.0)


# ------------------------------------------------------------------------------------------
# A3 enstrophy
# ------------------------------------------------------------------------------------------
ENS = dict(indicator="enstrophy", base_level=0, med_level=0, max_level=0, med_threshold=0.5, max_threshold=0.5)


def test_enstrophy_rigid_rotation():
    """v = Omega (-(y - y0), x - x0): w = 2 Omega, eps = 2 rho Omega^2 on every element (any size)"""
    lm = W.balance(np.kron(np.array([[2, 1], [1, 0]], np.uint8), np.ones((4, 4), np.uint8)), 2)
    m = _mesh(2, 2, lm)
    xy = m.node_coords()
    Om, rho = 1.7, 1.3
    U = _state(m, rho, -Om * (xy[:, 1] - 0.4), Om * (xy[:, 0] - 0.3), 2.0)
    assert len(set(m.leaves()["level"])) == 3
    assert np.allclose(m.amr_indicator(U, ENS), 2 * rho * Om * Om, rtol=1e-12)


def test_enstrophy_polynomial_field():
    """v_x = y^2, v_y = x^3: w = 3 x^2 - 2 y (exact for the cubic interpolant); max over nodes"""
    m = _mesh(2, 1, np.array([[1, 1, 0, 0], [1, 1, 0, 0], [0, 0, 0, 0], [0, 0, 0, 0]], np.uint8))
    xy = m.node_coords()
    x, y = xy[:, 0], xy[:, 1]
    rho = 0.8 + 0.1 * x
    U = _state(m, rho, y * y, x ** 3, 1.0)
    want = (0.5 * rho * (3 * x * x - 2 * y) ** 2).max(axis=1)
    assert np.allclose(m.amr_indicator(U, ENS), want, rtol=1e-11)


# ------------------------------------------------------------------------------------------
# A4-A6 controller and balance
# ------------------------------------------------------------------------------------------
CTRL = dict(indicator="enstrophy", base_level=0, med_level=1, max_level=2, med_threshold=1.0, max_threshold=10.0)
EPS_OF_TARGET = {0: 0.0, 1: 5.0, 2: 50.0}


def _state_with_targets(m, targets):
    """rigid rotation per element with eps = 2 Omega^2 (rho = 1) in the bucket of the target level"""
    xy = m.node_coords()
    Om = np.sqrt(np.array([EPS_OF_TARGET[t] for t in targets]) / 2.0)[:, None]
    return _state(m, 1.0, -Om * xy[:, 1], Om * xy[:, 0], 1.0)


def test_controller_coarsen_all():
    m = _mesh(2, 2, np.ones((8, 8), np.uint8))
    U = _state_with_targets(m, [0] * m.n)
    assert np.all(m.amr_adapt(U, CTRL) == 0)


def test_controller_sibling_veto_and_one_level_step():
    m = _mesh(2, 2, np.ones((8, 8), np.uint8))
    t = [0] * m.n
    t[5] = 1                                     # one child of the second base cell stays
    t[12] = 2                                    # a child of the fourth base cell wants level 2
    U = _state_with_targets(m, t)
    lm = m.amr_adapt(U, CTRL)
    lv = m.leaves()
    got = lm[lv["fy"], lv["fx"]]
    # base cell of leaf 5 (leaves 4..7) keeps level 1; leaf 12 -> level 2 (one step), its siblings keep 1;
    # base cell (0, 0) coarsens; base cell (0, 1) would coarsen but faces leaf 12's level-2 children
    # across x = 4, so the balance splits it again (level 1)
    assert all(got[k] == 1 for k in range(4, 8))
    assert got[12] == 2 and lm[lv["fy"][12]:lv["fy"][12] + 2, lv["fx"][12]:lv["fx"][12] + 2].min() == 2
    assert all(got[k] == 1 for k in (13, 14, 15))
    assert all(got[k] == 0 for k in range(0, 4)) and all(got[k] == 1 for k in range(8, 12))
    assert np.all(lm[0:4, 0:4] == 0)


def _all_trees(L):
    """every quadtree of depth <= L over one base cell, as (2^L x 2^L) level blocks"""
    s = 1 << L

    def rec(lev):
        n = 1 << (L - lev)
        out = [np.full((n, n), lev, np.uint8)]
        if lev < L:
            subs = rec(lev + 1)
            h = n // 2
            for a, b, c, d in itertools.product(subs, repeat=4):
                blk = np.empty((n, n), np.uint8)
                blk[:h, :h], blk[:h, h:], blk[h:, :h], blk[h:, h:] = a, b, c, d
                out.append(blk)
        return out
    trees = rec(0)
    assert all(t.shape == (s, s) for t in trees)
    return trees


def _balanced(lm, periodic):
    for ax in (0, 1):
        d = np.abs(lm.astype(int) - np.roll(lm, 1, axis=ax).astype(int))
        if not periodic[1 - ax]:
            d = d[1:] if ax == 0 else d[:, 1:]
        if d.max(initial=0) > 1:
            return False
    return True


def _min_balanced_brute(M0, nb, L, periodic):
    trees = _all_trees(L)
    s = 1 << L
    cand = []
    for by in range(nb):
        for bx in range(nb):
            blk = M0[by * s:(by + 1) * s, bx * s:(bx + 1) * s]
            cand.append([t for t in trees if np.all(t >= blk)])
    best, best_leaves = None, None
    for combo in itertools.product(*cand):
        lm = np.zeros_like(M0)
        for k, t in enumerate(combo):
            by, bx = divmod(k, nb)
            lm[by * s:(by + 1) * s, bx * s:(bx + 1) * s] = t
        if not _balanced(lm, periodic):
            continue
        leaves = int((4.0 ** lm.astype(np.float64)).sum())     # sum over finest cells of 4^l / 4^L * 4^L
        if best is None or leaves < best_leaves:
            best, best_leaves = lm, leaves
        elif leaves == best_leaves:
            assert np.array_equal(lm, best), "minimal balanced refinement must be unique"
    return best


def _rasterised_decision(m, targets):
    """controller decision per leaf by hand: one step, siblings must all coarsen"""
    lv = m.leaves()
    L = m.problem["max_level"]
    want = [min(l + 1, t) if t > l else (max(l - 1, t) if t < l else l) for l, t in zip(lv["level"], targets)]
    n_f = m.problem["n_base"][0] << L
    M0 = np.zeros((n_f, n_f), np.uint8)
    pos = {(int(x), int(y)): e for e, (x, y) in enumerate(zip(lv["fx"], lv["fy"]))}
    for e in range(m.n):
        l, s = int(lv["level"][e]), 1 << (L - int(lv["level"][e]))
        nl = want[e]
        if nl < l:
            px, py = lv["fx"][e] - lv["fx"][e] % (2 * s), lv["fy"][e] - lv["fy"][e] % (2 * s)
            for cy in (0, 1):
                for cx in (0, 1):
                    c = pos.get((int(px + cx * s), int(py + cy * s)))
                    if c is None or lv["level"][c] != l or want[c] >= l:
                        nl = l
        M0[lv["fy"][e]:lv["fy"][e] + s, lv["fx"][e]:lv["fx"][e] + s] = nl
    return M0


@pytest.mark.parametrize("periodic", [(1, 1), (0, 0), (1, 0)])
@pytest.mark.parametrize("seed", range(4))
def test_balance_is_minimal_brute_force(seed, periodic):
    rng = np.random.default_rng(seed)
    nb, L = 2, 2
    start = W.balance(rng.integers(0, 3, (nb << L, nb << L)).astype(np.uint8), L, periodic)
    m = _mesh(nb, L, start, periodic)
    targets = rng.integers(0, 3, m.n)
    lm = m.amr_adapt(_state_with_targets(m, targets), CTRL)
    want = _min_balanced_brute(_rasterised_decision(m, targets), nb, L, periodic)
    assert np.array_equal(lm, want)


@pytest.mark.parametrize("seed", range(3))
def test_balance_matches_generator_balance(seed):
    """larger meshes: the oracle's leaf-splitting fixpoint == the generator's independent
    neighbour-max / leafify iteration (workloads.balance) applied to the controller decision"""
    rng = np.random.default_rng(10 + seed)
    nb, L = 6, 3
    start = W.balance(rng.integers(0, 4, (nb << L, nb << L)).astype(np.uint8), L)
    m = _mesh(nb, L, start)
    ctrl = dict(CTRL, max_level=3)
    eps = {0: 0.0, 1: 5.0, 3: 50.0}
    targets = rng.choice([0, 1, 3], m.n)
    xy = m.node_coords()
    Om = np.sqrt(np.array([eps[t] for t in targets]) / 2.0)[:, None]
    U = _state(m, 1.0, -Om * xy[:, 1], Om * xy[:, 0], 1.0)
    lm = m.amr_adapt(U, ctrl)
    assert np.array_equal(lm, W.balance(_rasterised_decision(m, targets), L))
    assert _balanced(lm, (1, 1))


def test_amr_rejects_bad_parameters():
    m = _mesh()
    U = _state(m, 1.0, 0.0, 0.0, 1.0)
    with pytest.raises(ValueError):
        m.amr_indicator(U, dict(CTRL, max_level=5))
    with pytest.raises(ValueError):
        m.amr_indicator(U, dict(CTRL, med_threshold=20.0))


def test_controller_one_level_per_adaptation_from_base():
    """a base-level leaf whose indicator asks for max_level (2) moves one level only (A4)"""
    m = _mesh(2, 2, np.zeros((8, 8), np.uint8))
    t = [0] * m.n
    t[3] = 2
    lm = m.amr_adapt(_state_with_targets(m, t), CTRL)
    lv = m.leaves()
    blk = lm[lv["fy"][3]:lv["fy"][3] + 4, lv["fx"][3]:lv["fx"][3] + 4]
    assert np.all(blk == 1)
    assert int(lm.max()) == 1


def test_controller_threshold_is_inclusive():
    """target = base level if indicator <= med_threshold (A4): a leaf whose indicator EQUALS the
    threshold coarsens with its siblings; just above it, it keeps the block refined"""
    m = _mesh(2, 2, np.ones((8, 8), np.uint8))
    t = [0] * m.n
    t[0] = 1
    U = _state_with_targets(m, t)
    ind = m.amr_indicator(U, CTRL)
    at = dict(CTRL, med_threshold=float(ind[0]))
    assert np.all(m.amr_adapt(U, at)[0:4, 0:4] == 0)
    below = dict(CTRL, med_threshold=float(np.nextafter(ind[0], 0.0)))
    assert np.all(m.amr_adapt(U, below)[0:4, 0:4] == 1)


def test_controller_on_given_indicator_equals_adapt():
    """ora_amr_adapt_ind (the controller + balance on given indicator values, used by the GPU map
    comparison) is ora_amr_adapt without the indicator pass"""
    m = _mesh(2, 2, np.ones((8, 8), np.uint8))
    t = [0] * m.n
    t[5], t[12] = 1, 2
    U = _state_with_targets(m, t)
    ind = m.amr_indicator(U, CTRL)
    assert np.array_equal(m.amr_adapt(None, CTRL, indicator=ind), m.amr_adapt(U, CTRL))
    flipped = ind.copy()
    flipped[12] = 0.0                            # leaf 12 wants to coarsen like its siblings
    lm = m.amr_adapt(None, CTRL, indicator=flipped)
    lv = m.leaves()
    assert m.amr_adapt(U, CTRL)[lv["fy"][12], lv["fx"][12]] == 2
    assert lm[lv["fy"][12], lv["fx"][12]] == 0
