"""Pins of the oracle's DGSEM basis and 1D weak-form operators and of the
partitioned P-ERK step on the DG system (O4): exact solutions, conservation, the cfg-2
contact-wave invariant, single-level reduction, temporal order, reference == restricted."""
import numpy as np
import pytest
import scipy.linalg

import workloads as W
from oracle import oracle as O
from oracle import tableau as T


def test_lgl_basis_facts():
    b = O.basis()
    xi, w, D = b["xi"], b["w"], b["D"]
    assert abs(w.sum() - 2.0) < 1e-15
    for k in range(6):   # LGL 4-point quadrature is exact to degree 2N-1 = 5
        assert abs((w * xi ** k).sum() - (2.0 / (k + 1) if k % 2 == 0 else 0.0)) < 1e-15
    assert np.abs(D @ np.ones(4)).max() < 1e-14
    for k in range(1, 4):  # exact on cubics
        assert np.abs(D @ xi ** k - k * xi ** (k - 1)).max() < 1e-13
    # closed form of D
    s5 = np.sqrt(5.0)
    D0 = [-3, (5 + 5 * s5) / 4, (5 - 5 * s5) / 4, 0.5]
    assert np.abs(D[0] - D0).max() < 1e-14
    # SBP: W D + (W D)^T = diag(-1, 0, 0, 1)
    Q = np.diag(w) @ D
    assert np.abs(Q + Q.T - np.diag([-1, 0, 0, 1])).max() < 1e-14
    # Dsplit has a vanishing diagonal for LGL N=3
    assert np.abs(np.diag(b["Dsplit"])).max() < 1e-14


def test_mortar_operators():
    b = O.basis()
    xi, w = b["xi"], b["w"]
    one = np.ones(4)
    for P in (b["Plo"], b["Pup"]):
        assert np.abs(P @ one - 1).max() < 1e-15
    assert np.abs((b["Rlo"] + b["Rup"]) @ one - 1).max() < 1e-14   # projection of a constant
    for R in (b["Rlo"], b["Rup"]):
        assert np.abs(w @ R - 0.5 * w).max() < 1e-15          # conservation
    assert np.abs(b["Rlo"] @ b["Plo"] + b["Rup"] @ b["Pup"] - np.eye(4)).max() < 1e-13  # coarsen o refine = I
    for k in range(4):   # interpolation exact for cubics
        p = xi ** k
        assert np.abs(b["Plo"] @ p - ((xi - 1) / 2) ** k).max() < 1e-14
        assert np.abs(b["Pup"] @ p - ((xi + 1) / 2) ** k).max() < 1e-14
        # projection of a global cubic restricted to the halves gives it back
        assert np.abs(b["Rlo"] @ (((xi - 1) / 2) ** k) + b["Rup"] @ (((xi + 1) / 2) ** k) - p).max() < 1e-13


def _assemble(m):
    nd = m.n * m.nv * m.npe
    L = np.zeros((nd, nd))
    for j in range(nd):
        e = np.zeros(nd)
        e[j] = 1.0
        L[:, j] = m.rhs(e.reshape(m.shape)).ravel()
    return L


def _mass(m, U):
    """sum_e (h/2) sum_i w_i U_i per variable."""
    w = O.basis()["w"]
    lev = m.leaves()["level"].astype(float)
    p = m.problem
    h = (p["domain_hi"][0] - p["domain_lo"][0]) / (p["n_base"][0] * 2.0 ** lev)
    return np.einsum("e,evi,i->v", h / 2, U, w)


@pytest.fixture(scope="module")
def cfg1():
    w = W.make(1)
    fam = T.family(w.S, w.E, "taylor")
    return w, fam, O.OracleMesh(w.problem, w.level_map, fam)


def test_cfg1_mesh(cfg1):
    w, fam, m = cfg1
    assert m.n == 48 and m.face_counts()["interfaces"] == 48
    assert list(m.count_active("elements")) == [48, 32, 32, 32, 32, 48, 48, 48]


def test_cfg1_energy_stable_spectrum(cfg1):
    w, fam, m = cfg1
    lam = np.linalg.eigvals(_assemble(m))
    assert lam.real.max() <= 1e-13 * np.abs(lam).max()


def test_cfg1_exact_solution(cfg1):
    """200 steps at CFL 0.2: vs exp(T L) U0 (time-integration error) and vs u0(x - T) (spatial)."""
    w, fam, m = cfg1
    U0 = m.initial_state(w.ic)
    U = U0.copy()
    ev = m.step(U, w.dt, w.steps)
    assert ev == 320 * w.steps          # sum_r E_r N_C(r) per step (P:l.1282-1289)
    Tend = w.dt * w.steps
    ex = (scipy.linalg.expm(Tend * _assemble(m)) @ U0.ravel()).reshape(U.shape)
    assert np.abs(U - ex).max() < 5e-8
    xs = m.node_coords()
    exact = w.ic(((xs - Tend) + 1.0) % 2.0 - 1.0)[0]
    assert np.abs(U[:, 0, :] - exact).max() < 1e-4
    m0, m1 = _mass(m, U0), _mass(m, U)
    assert abs(m1 - m0).max() <= 1e-14 * np.abs(_mass(m, np.abs(U0))).max() * 10


def test_reference_equals_restricted(cfg1):
    w, fam, m = cfg1
    U0 = m.initial_state(w.ic)
    a, b = U0.copy(), U0.copy()
    m.step(a, w.dt, 3, mode=0)
    m.step(b, w.dt, 3, mode=1)
    assert np.array_equal(a, b)
    for mask in (2, 3):      # upward-closed masks (the ones P-ERK stages use)
        assert np.array_equal(m.rhs(U0, mask, 0), m.rhs(U0, mask, 1))
    with pytest.raises(ValueError):
        m.rhs(U0, 1, 1)


def test_single_level_reduction_dg():
    """All cells at the finest level: multirate family == single-rate S-stage P-ERK, bitwise."""
    w = W.make(2, n_base=32, w1=16, w2=4)
    lm = np.full_like(w.level_map, w.problem["max_level"])
    famR = T.family(16, [4, 8, 16], "taylor")
    fam1 = T.family(16, [16], "taylor")
    mR = O.OracleMesh(w.problem, lm, famR)
    p1 = dict(w.problem, max_level=w.problem["max_level"])
    m1 = O.OracleMesh(p1, lm, fam1)
    U0 = mR.initial_state(w.ic)
    a, b = U0.copy(), U0.copy()
    mR.step(a, w.dt, 5)
    m1.step(b, w.dt, 5)
    assert np.array_equal(a, b)


@pytest.fixture(scope="module")
def cfg2_run():
    w = W.make(2)
    fam = T.family(w.S, w.E, "taylor")
    m = O.OracleMesh(w.problem, w.level_map, fam)
    U0 = m.initial_state(w.ic)
    U = U0.copy()
    ev = m.step(U, w.dt, w.steps)
    return w, m, U0, U, ev


def test_cfg2_contact_invariant(cfg2_run):
    """Euler with v = 1, p = 1 is a contact wave: v and p stay 1."""
    w, m, U0, U, ev = cfg2_run
    assert m.n == 352 and ev == 2560 * w.steps
    rho, mom, E = U[:, 0], U[:, 1], U[:, 2]
    v = mom / rho
    p = 0.4 * (E - 0.5 * rho * v * v)
    assert np.abs(v - 1).max() < 1e-13 and np.abs(p - 1).max() < 1e-13
    xs = m.node_coords()
    Tend = w.dt * w.steps
    assert np.abs(rho - w.ic(((xs - Tend) % 2.0))[0]).max() < 1e-7
    for v_ in range(3):
        m0, m1 = _mass(m, U0)[v_], _mass(m, U)[v_]
        assert abs(m1 - m0) <= 1e-14 * abs(m0) * 10


def test_temporal_order_dg_euler():
    """dt-halving against a 16x finer reference, 1D Euler cfg-2 mesh with a nonlinear IC: order >= 1.9."""
    w = W.make(2, n_base=64, w1=16, w2=4)
    fam = T.family(w.S, w.E, "taylor")
    m = O.OracleMesh(w.problem, w.level_map, fam)

    def ic(x):
        rho = 1 + 0.3 * np.sin(np.pi * x)
        v = 1 + 0.3 * np.cos(np.pi * x)
        p = 1 + 0.3 * np.sin(np.pi * x + 1)
        return np.stack([rho, rho * v, p / 0.4 + 0.5 * rho * v * v])

    U0 = m.initial_state(ic)
    dt0 = 8 * w.dt
    Tend = 8 * dt0

    def run(dt):
        U = U0.copy()
        m.step(U, dt, int(round(Tend / dt)))
        return U

    ref = run(dt0 / 64)
    errs = [np.abs(run(dt0 / 2 ** k) - ref).max() for k in range(3)]
    orders = [np.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert min(orders) >= 1.9, orders
