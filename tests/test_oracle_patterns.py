"""Stage-pattern variants and alternative weights (oracle/tableau.py; F1-F3),
pinned against the paper and the mathematics:

* the printed S = 6, E = 4 tableaux: standard (P:l.410-420), alternating (P:l.655-675) and
  early-shared (P:l.683-700): evaluated stages and the positions of every nonzero a_{i,j};
* every pattern / weight choice: b^T 1 = 1, b^T c = 1/2, internal consistency, and the member's
  stability polynomial b^T A^(k-1) 1 = alpha_k (k <= E), 0 beyond, by exact matrix powers of the
  dense Butcher matrix (P:l.1040-1064);
* S = 2 reduces to Heun's and Ralston's methods (P:l.439-442, textbook tableaux);
* the oracle's step with one member equals P(dt L) U on a linear system (brute force) for every
  pattern; with several members and NON-nested patterns it equals a brute-force dense partitioned
  Runge-Kutta step (P:l.209-218, all K_j stored) on the nonlinear Burgers testbed;
* conservation and second-order convergence with patterns; the DG oracle's restricted mode falls
  back to the definition for the non-upward-closed stage masks these patterns produce.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from oracle import tableau as T
from test_oracle_fv import _cell_avg_ic, _mesh


def _printed_nonzeros(A):
    """positions (i, j), 1-based, of the nonzero entries right of the first column"""
    return sorted((i + 1, j + 1) for i, row in enumerate(A) for j, v in enumerate(row) if j > 0 and v != 0)


@pytest.mark.parametrize("pattern,stages,nonzeros", [
    ("standard", [1, 4, 5, 6], [(5, 4), (6, 5)]),          # P:l.410-420, A^(1)
    ("alternating", [1, 3, 4, 6], [(4, 3), (6, 4)]),       # P:l.655-675
    ("early", [1, 2, 3, 6], [(3, 2), (6, 3)]),             # P:l.683-700
])
def test_printed_s6_tableaux(pattern, stages, nonzeros):
    fam = T.family(6, [4, 6], "taylor", pattern=pattern)
    assert fam["c"] == [Fr(i, 10) for i in range(6)]
    assert fam["stages"][0] == stages
    A = T.butcher(fam, 0)
    assert _printed_nonzeros(A) == nonzeros
    for i in range(6):                                      # first column c_i - a_{i,p(i)}
        assert sum(A[i]) == fam["c"][i]
    # the E = S member evaluates every stage and has a_{i,i-1} for i >= 3 (P:l.410-420, A^(2))
    assert fam["stages"][1] == [1, 2, 3, 4, 5, 6]
    assert _printed_nonzeros(T.butcher(fam, 1)) == [(3, 2), (4, 3), (5, 4), (6, 5)]


def _poly_coeffs(fam, r, kmax):
    S = fam["S"]
    A = T.butcher(fam, r)
    b = fam["b"]
    v = [Fr(1)] * S
    out = []
    for k in range(1, kmax + 1):
        out.append(sum(bi * vi for bi, vi in zip(b, v)))        # b^T A^(k-1) 1
        v = [sum(A[i][j] * v[j] for j in range(S)) for i in range(S)]
    return out


@pytest.mark.parametrize("S,Es", [(6, [2, 3, 4, 6]), (8, [3, 4, 8]), (16, [4, 8, 16]), (12, [5, 7, 12])])
@pytest.mark.parametrize("pattern", ["standard", "alternating", "early"])
@pytest.mark.parametrize("c_S", [Fr(1, 2), Fr(1), Fr(2, 3)])
def test_polynomial_and_order_conditions(S, Es, pattern, c_S):
    fam = T.family(S, Es, "taylor", pattern=pattern, c_S=c_S)
    b, c = fam["b"], fam["c"]
    assert sum(b) == 1 and sum(bi * ci for bi, ci in zip(b, c)) == Fr(1, 2)       # P:l.236-237
    assert c[-1] == c_S and b[-1] == 1 / (2 * c_S)
    for r, E in enumerate(Es):
        coef = _poly_coeffs(fam, r, S + 1)
        for k in range(1, S + 2):
            want = fam["alpha"][r][k] if k <= E else 0
            assert coef[k - 1] == want, (pattern, E, k)
        A = T.butcher(fam, r)
        for i in range(S):
            assert sum(A[i]) == c[i]                                              # internal consistency
            nz = [j for j in range(1, S) if A[i][j] != 0]
            assert len(nz) <= 1                                                   # two nonzeros per row


def test_heun_ralston_at_s2():
    """S = 2: c_S = 1 is Heun's method, c_S = 2/3 Ralston's (P:l.439-442)"""
    h = T.family(2, [2], c_S=1)
    assert h["c"] == [0, 1] and h["b"] == [Fr(1, 2), Fr(1, 2)] and T.butcher(h, 0) == [[0, 0], [1, 0]]
    r = T.family(2, [2], c_S=Fr(2, 3))
    assert r["c"] == [0, Fr(2, 3)] and r["b"] == [Fr(1, 4), Fr(3, 4)]
    assert T.butcher(r, 0) == [[0, 0], [Fr(2, 3), 0]]
    m = T.family(2, [2])                                    # the standard choice: explicit midpoint
    assert m["b"] == [0, 1] and T.butcher(m, 0) == [[0, 0], [Fr(1, 2), 0]]


def _fv_matrix(dx):
    n = len(dx)
    L = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        L[:, j] = O.fv_rhs(dx, e, kind=0)
    return L


@pytest.mark.parametrize("pattern", ["alternating", "early", [1, 2, 5, 7, 8]])
@pytest.mark.parametrize("c_S", [Fr(1, 2), Fr(1), Fr(2, 3)])
def test_single_member_step_is_polynomial(pattern, c_S):
    S, E = 8, 5
    dx = np.full(24, 2.0 / 24)
    fam = T.family(S, [E], pattern=pattern, c_S=c_S)
    x = np.cumsum(dx)
    U0 = np.sin(np.pi * x) + 0.4 * np.cos(3 * np.pi * x)
    dt = 0.4 * dx[0]
    got = O.fv_step(dx, np.zeros(24, np.int32), fam, U0, dt)
    Z = dt * _fv_matrix(dx)
    want, term = np.zeros_like(U0), U0.copy()
    for k in range(E + 1):
        want += float(fam["alpha"][0][k]) * term
        term = Z @ term
    assert np.abs(got - want).max() <= 1e-13 * np.abs(U0).max()


def _burgers(U, dx):
    return O.fv_rhs(dx, U, kind=1)


def _dense_partitioned_step(dx, mem, fam, U, dt):
    """P:l.209-218 literally: K_j^(r) = I^(r) F(U_n + dt sum_k sum_l a_{jl}^(k) K_l^(k)), all K stored"""
    S, R = fam["S"], fam["R"]
    A = [[[float(v) for v in row] for row in T.butcher(fam, r)] for r in range(R)]
    b = [float(v) for v in fam["b"]]
    K = []
    for i in range(S):
        Ui = U.copy()
        for j in range(i):
            for r in range(R):
                sel = mem == r
                Ui[sel] += dt * A[r][i][j] * K[j][sel]
        F = _burgers(Ui, dx)
        Ki = np.zeros_like(U)
        for r in range(R):
            if (i + 1) in fam["stages"][r]:
                Ki[mem == r] = F[mem == r]
        K.append(Ki)
    return U + dt * sum(b[i] * K[i] for i in range(S))


@pytest.mark.parametrize("c_S", [Fr(1, 2), Fr(1)])
def test_non_nested_patterns_equal_dense_partitioned_rk(c_S):
    """three members whose evaluated-stage sets are not nested"""
    S = 8
    pats = [[1, 3, 6, 8], [1, 2, 4, 5, 8], [1, 2, 3, 4, 5, 6, 7, 8]]
    fam = T.family(S, [4, 5, 8], pattern=pats, c_S=c_S)
    assert fam["active_mask"] is not None
    n = 36
    dx = np.full(n, 2.0 / n)
    mem = np.repeat(np.array([0, 1, 2, 1, 0, 2], np.int32), 6)
    U0 = _cell_avg_ic(dx)
    dt = 0.05 * dx[0]
    U = U0.copy()
    Ud = U0.copy()
    for _ in range(5):
        U = O.fv_step(dx, mem, fam, U, dt, kind=1)
        Ud = _dense_partitioned_step(dx, mem, fam, Ud, dt)
    assert np.abs(U - Ud).max() <= 1e-14 * np.abs(U0).max()
    assert abs(np.sum(U * dx) - np.sum(U0 * dx)) <= 1e-14                       # conservation


@pytest.mark.parametrize("pattern", ["alternating", "early"])
def test_burgers_second_order_patterns(pattern):
    dx, mem = _mesh(64)
    fam = T.family(16, [8, 16], pattern=pattern)
    U0 = _cell_avg_ic(dx)
    Tend = 0.25

    def run(nsteps):
        U = U0.copy()
        for _ in range(nsteps):
            U = O.fv_step(dx, mem, fam, U, Tend / nsteps, kind=1)
        return U

    ref = run(1280)
    errs = [np.abs(run(n) - ref).max() for n in (40, 80, 160)]
    orders = [np.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert all(1.85 < o < 2.3 for o in orders), orders


def test_dg_patterns_restricted_fallback_and_conservation():
    """2D DG with non-nested stage masks: restricted mode (fallback to the definition for masks
    that are not upward closed) == reference mode bitwise; conservation"""
    w = W.make(3, n_base=8)
    fam = T.family(16, [4, 8, 16], pattern=[[1, 5, 9, 16], [1, 2, 4, 6, 8, 10, 12, 16], "standard"])
    m1 = O.OracleMesh(w.problem, w.level_map, fam)
    m0 = O.OracleMesh(w.problem, w.level_map, fam)
    U1 = m1.initial_state(w.ic)
    U0 = U1.copy()
    tot0 = U1.sum(axis=(0, 2))
    m1.step(U1, w.dt, 3, mode=1)
    m0.step(U0, w.dt, 3, mode=0)
    assert np.array_equal(U1, U0)
    lv = m1.leaves()["level"]
    b = O.basis()
    h = 10.0 / (8 * 4) * 2.0 ** (2 - lv.astype(np.float64))
    wq = np.outer(b["w"], b["w"]).ravel()

    def totals(U):
        return np.array([np.sum((h[:, None] / 2) ** 2 * wq[None, :] * U[:, v, :]) for v in range(4)])
    Ui = m1.initial_state(w.ic)
    assert np.all(np.abs(totals(U1) - totals(Ui)) <= 1e-13 * np.abs(totals(Ui)).max())
    del tot0
