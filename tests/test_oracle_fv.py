"""Pins of the oracle's partitioned P-ERK stepper against the paper's Godunov FV example
(§3.2, l.479-815): spectrum of D, negative entries of D, row sums, the
printed total-variation tables, conservation and second-order convergence."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import tableau as T

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _mesh(N1, alpha=2):
    """coarse dx = 2/N1 on (-1,-0.5) u (0.5,1), dx/alpha on [-0.5,0.5]; member 1 = refined."""
    dxc = 2.0 / N1
    nc = N1 // 4
    nf = int(round(alpha * N1 / 2))
    dx = np.concatenate([np.full(nc, dxc), np.full(nf, 1.0 / nf), np.full(nc, dxc)])
    mem = np.concatenate([np.zeros(nc), np.ones(nf), np.zeros(nc)]).astype(np.int32)
    return dx, mem


def _cell_avg_ic(dx):
    """exact cell averages of u0 = 1 + sin(pi x)/2 (eq. 1DAdvection)."""
    xr = -1.0 + np.cumsum(dx)
    xl = xr - dx
    return 1.0 + (np.cos(np.pi * xl) - np.cos(np.pi * xr)) / (2 * np.pi * dx)


def _tv(U):
    return np.abs(np.roll(U, -1) - U).sum()  # periodic wrap included


def _D(dx, mem, fam, dt):
    n = len(dx)
    D = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        D[:, j] = O.fv_step(dx, mem, fam, e, dt)
    return D


@pytest.fixture(scope="module")
def uniform_D():
    """uniform N = 64, E = 16 in [-0.5, 0.5], E = 8 elsewhere, dt = 0.21875 (l.535-569)."""
    dx = np.full(64, 2.0 / 64)
    xc = -1.0 + (np.arange(64) + 0.5) * 2.0 / 64
    mem = ((xc > -0.5) & (xc < 0.5)).astype(np.int32)
    fam = T.family(16, [8, 16], "disk")
    return _D(dx, mem, fam, 0.21875), mem


def test_spectral_radius_uniform(uniform_D):
    """rho(D) <= 1 with the conservation eigenvalue 1 (l.568, caption l.578)."""
    D, _ = uniform_D
    lam = np.linalg.eigvals(D)
    k = np.argmin(np.abs(lam - 1.0))
    assert abs(lam[k] - 1.0) < 1e-13
    rest = np.delete(np.abs(lam), k)
    assert rest.max() < 1.0


def test_row_sums_one(uniform_D):
    """each row sum d_i = 1: conservation (l.631)."""
    D, _ = uniform_D
    assert np.abs(D.sum(axis=1) - 1.0).max() < 1e-12


def test_negative_rows_17_24(uniform_D):
    """rows i = 17..24 (1-based) of D have negative entries (l.619-622)."""
    D, mem = uniform_D
    for i in range(17, 25):
        assert D[i - 1].min() < -1e-6, i
    # the first member-1 cells are 17..48 (1-based): the loss of monotonicity sits at the
    # left (upwind) transition where the E=16 method reads first-order E=8 data
    assert mem[16] == 1 and mem[15] == 0


def _tv_case(kind, p):
    if kind == "cfl":
        dx, mem = _mesh(64)
        fam = T.family(16, [8, 16], "disk")
        dt = p * 0.21875
    elif kind == "n":
        dx, mem = _mesh(int(p))
        fam = T.family(16, [8, 16], "disk")
        dt = 7 * 2.0 / p
    else:
        E1 = int(p)
        dx, mem = _mesh(64)
        fam = T.family(2 * E1, [E1, 2 * E1], "disk")
        dt = (E1 - 1) * 2.0 / 64
    U0 = _cell_avg_ic(dx)
    U1 = O.fv_step(dx, mem, fam, U0, dt)
    return (_tv(U1) - _tv(U0)) / _tv(U0)


def _tv_rows():
    rows = []
    for line in open(os.path.join(GOLD, "tv_tables.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, p, v, tol = line.split()
        rows.append((k, float(p), float(v), float(tol)))
    return rows


@pytest.mark.parametrize("kind,p,printed,tol", _tv_rows())
def test_tv_tables(kind, p, printed, tol):
    assert abs(_tv_case(kind, p) - printed) <= tol


def test_conservation_fv():
    dx, mem = _mesh(64)
    fam = T.family(16, [8, 16], "disk")
    U = _cell_avg_ic(dx)
    m0 = (dx * U).sum()
    for _ in range(20):
        U = O.fv_step(dx, mem, fam, U, 0.1)
    assert abs((dx * U).sum() - m0) <= 1e-14 * abs(m0) * 20


def test_burgers_second_order():
    """Burgers FV testbed, 2 levels, Taylor {4, 8}: temporal order 2 (l.632)."""
    dx, mem = _mesh(64)
    fam = T.family(8, [4, 8], "taylor")
    U0 = _cell_avg_ic(dx)
    Tend = 0.25

    def run(nsteps):
        U = U0.copy()
        for _ in range(nsteps):
            U = O.fv_step(dx, mem, fam, U, Tend / nsteps, kind=1)
        return U

    ref = run(640)
    errs = [np.abs(run(n) - ref).max() for n in (10, 20, 40)]
    orders = [np.log2(errs[k] / errs[k + 1]) for k in range(2)]
    for o in orders:
        assert abs(o - 2.0) < 0.05, orders


def test_single_member_reduces_to_rk_polynomial_on_burgers():
    """All cells in the E = S member: the family's step equals the single-rate S-stage method bitwise."""
    dx, _ = _mesh(64)
    famR = T.family(16, [8, 16], "disk")
    fam1 = T.family(16, [16], "disk")
    U0 = _cell_avg_ic(dx)
    a = O.fv_step(dx, np.ones(len(dx), np.int32), famR, U0, 0.05, kind=1)
    b = O.fv_step(dx, np.zeros(len(dx), np.int32), fam1, U0, 0.05, kind=1)
    assert np.array_equal(a, b)
