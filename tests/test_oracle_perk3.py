"""P-ERK3: the generated families (workloads/perk3.py, reading P3b) checked against
the paper's conditions, and the oracle's general-b stepper pinned on them.

* every family: b^T 1 = 1, b^T c = 1/2, b^T c^2 = 1/3 (exact), b^T A^(r) c = 1/6 for every member
  (P:l.236-240, eq. PRKOrderCondsSimplified; P:l.1085) and the member's stability polynomial
  b^T A^(k-1) 1 = alpha_k = 1/k! for 4 <= k <= E, 0 beyond (P:l.1040-1042, l.1072-1080), computed by
  explicit matrix powers in 80-digit arithmetic, not by the generator's chain formula; positivity
  of a_{i,i-1} and a_{i,1} (P:l.1088-1089);
* the E = 3 member is the Shu-Osher SSPRK3 tableau (P:l.870-880);
* the oracle's step with a single member equals P(dt L) U on a linear FV system (brute force);
* temporal order 3 on the Burgers FV testbed and >= 2.9 on a nonlinear DG Euler problem with two and
  three members; conservation; single-level reduction (bitwise).
"""
import mpmath as mp
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from test_oracle_fv import _cell_avg_ic, _mesh
from workloads import perk3 as P3

FAMS = [(8, (3, 4, 8)), (12, (3, 6, 12)), (16, (4, 8, 16)), (32, (4, 8, 16, 32))]


def _A_mp(S, c, x):
    A = mp.zeros(S, S)
    for i in range(2, S + 1):
        xi = x.get(i, mp.mpf(0))
        A[i - 1, i - 2] += xi
        A[i - 1, 0] += mp.mpf(c[i - 1].numerator) / c[i - 1].denominator - xi
    return A


@pytest.mark.parametrize("S,Es", FAMS)
def test_family_order_conditions_and_polynomial(S, Es):
    fam = P3.family3(S, Es)
    c, b = fam["c"], fam["b"]
    assert sum(b) == 1
    assert sum(bi * ci for bi, ci in zip(b, c)) * 2 == 1
    assert sum(bi * ci * ci for bi, ci in zip(b, c)) * 3 == 1
    with mp.workdps(80):
        bv = mp.matrix([mp.mpf(v.numerator) / v.denominator for v in b]).T
        one = mp.matrix([1] * S)
        for r, E in enumerate(Es):
            x = fam["asub_mp"][r]
            A = _A_mp(S, c, x)
            cv = A * one
            assert mp.fabs((bv * A * cv)[0] - mp.mpf(1) / 6) < mp.mpf(10) ** -60
            v = one
            for k in range(1, S + 1):
                coef = (bv * v)[0]                    # b^T A^(k-1) 1
                want = mp.mpf(1) / mp.factorial(k) if k <= E else mp.mpf(0)
                # relative to 1/k!: the generated roots carry >= 50 correct digits (3.7e-51 at E = 32)
                assert mp.fabs(coef - want) <= mp.mpf(10) ** -45 / mp.factorial(k), (E, k)
                v = A * v
            for i in range(1, S + 1):
                xi = x.get(i, mp.mpf(0))
                ci = mp.mpf(c[i - 1].numerator) / c[i - 1].denominator
                assert xi >= 0 and ci - xi >= 0 and (i == 1 or ci - xi > 0 or ci == 0), (E, i)
            # the rounded doubles satisfy the third-order condition to rounding
            Ad = np.zeros((S, S))
            for i in range(2, S + 1):
                Ad[i - 1, i - 2] = fam["asub_f"][r][i - 1]
                Ad[i - 1, 0] = fam["a1_f"][r][i - 1]
            cd = np.array(fam["c_f"])
            assert abs(np.array(fam["b_f"]) @ Ad @ cd - 1 / 6) < 1e-15


def test_S3_is_shu_osher_ssprk3():
    """S = E = 3: the Shu-Osher base of P:l.870-880 (c = (0, 1, 1/2), a_21 = 1, a_31 = a_32 = 1/4,
    b = (1/6, 1/6, 4/6)) -- also SPEC.md's tableau example"""
    fam = P3.family3(3, (3,))
    assert fam["c_f"] == [0.0, 1.0, 0.5] and fam["b_f"] == [1 / 6, 1 / 6, 4 / 6]
    assert fam["a1_f"][0] == [0.0, 1.0, 0.25] and fam["asub_f"][0] == [0.0, 0.0, 0.25]


def test_E3_member_is_shu_osher():
    for S in (4, 8, 16):
        fam = P3.family3(S, (3,))
        a1, asub = fam["a1_f"][0], fam["asub_f"][0]
        assert fam["c_f"][S - 2] == 1.0 and fam["c_f"][S - 1] == 0.5
        assert a1[S - 2] == 1.0 and asub[S - 2] == 0.0                    # stage S-1: U_n + dt K_1
        assert a1[S - 1] == 0.25 and asub[S - 1] == 0.25                  # stage S: 1/4 K_1 + 1/4 K_{S-1}
        assert fam["b_f"][0] == 1 / 6 and fam["b_f"][S - 2] == 1 / 6 and fam["b_f"][S - 1] == 4 / 6
        for i in range(1, S - 2):
            assert asub[i] == 0.0                                          # inactive stages


def _fv_matrix(dx):
    n = len(dx)
    L = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        L[:, j] = O.fv_rhs(dx, e, kind=0)
    return L


@pytest.mark.parametrize("S,E", [(8, 3), (8, 8), (12, 6), (16, 16)])
def test_single_member_step_is_stability_polynomial(S, E):
    """one member on a uniform linear FV system: step(U) = sum_k alpha_k (dt L)^k U (matrix powers)"""
    dx = np.full(32, 2.0 / 32)
    mem = np.zeros(32, np.int32)
    fam = P3.family3(S, (E,))
    U0 = np.sin(np.pi * np.cumsum(dx)) + 0.3 * np.cos(3 * np.pi * np.cumsum(dx))
    dt = 0.5 * dx[0]
    got = O.fv_step(dx, mem, fam, U0, dt)
    Z = dt * _fv_matrix(dx)
    want = np.zeros_like(U0)
    term = U0.copy()
    for k in range(0, E + 1):
        alpha = 1.0 / float(mp.factorial(k))
        want += alpha * term
        term = Z @ term
    assert np.abs(got - want).max() <= 1e-13 * np.abs(U0).max()


def test_burgers_third_order():
    """Burgers FV testbed, 2 levels, P-ERK3 {4, 8}: temporal order 3"""
    dx, mem = _mesh(64)
    fam = P3.family3(8, (4, 8))
    U0 = _cell_avg_ic(dx)
    Tend = 0.25

    def run(nsteps):
        U = U0.copy()
        for _ in range(nsteps):
            U = O.fv_step(dx, mem, fam, U, Tend / nsteps, kind=1)
        return U

    ref = run(2560)
    errs = [np.abs(run(n) - ref).max() for n in (20, 40, 80, 160)]
    orders = [np.log2(errs[k] / errs[k + 1]) for k in range(3)]
    # observed 3.26, 3.14, 3.08: the Taylor polynomial's higher-order terms fade, order -> 3
    assert all(b < a for a, b in zip(orders, orders[1:])), orders
    assert 2.95 < orders[-1] < 3.12, orders


def _euler_p3_mesh():
    w = W.make(2, n_base=64, w1=16, w2=4)
    fam = P3.family3(12, (3, 6, 12))
    return w, fam, O.OracleMesh(w.problem, w.level_map, fam)


def _nonlinear_ic(x):
    rho = 1 + 0.3 * np.sin(np.pi * x)
    v = 1 + 0.3 * np.cos(np.pi * x)
    p = 1 + 0.3 * np.sin(np.pi * x + 1)
    return np.stack([rho, rho * v, p / 0.4 + 0.5 * rho * v * v])


def test_dg_euler_order_p3():
    w, fam, m = _euler_p3_mesh()
    U0 = m.initial_state(_nonlinear_ic)
    dt0 = 8 * w.dt
    Tend = 8 * dt0

    def run(dt):
        U = U0.copy()
        m.step(U, dt, int(round(Tend / dt)))
        return U

    ref = run(dt0 / 64)
    errs = [np.abs(run(dt0 / 2 ** k) - ref).max() for k in range(3)]
    orders = [np.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert min(orders) >= 2.9, orders


def test_dg_euler_conservation_p3():
    w, fam, m = _euler_p3_mesh()
    U = m.initial_state(_nonlinear_ic)
    b = O.basis()
    h = (w.problem["domain_hi"][0] - w.problem["domain_lo"][0]) / (w.problem["n_base"][0] * 4) * \
        2.0 ** (2 - m.leaves()["level"].astype(np.float64))
    def totals(U):
        return np.array([np.sum(h[:, None] / 2 * b["w"][None, :] * U[:, v, :]) for v in range(3)])
    t0 = totals(U)
    m.step(U, w.dt, 50)
    assert np.all(np.abs(totals(U) - t0) <= 1e-14 * np.abs(t0) * 50)


def test_single_level_reduction_p3():
    w = W.make(2, n_base=32, w1=8, w2=4)
    lm = np.full_like(w.level_map, w.problem["max_level"])
    multi = O.OracleMesh(w.problem, lm, P3.family3(12, (3, 6, 12)))
    single = O.OracleMesh(w.problem, lm, P3.family3(12, (12,)))
    Ua = multi.initial_state(_nonlinear_ic)
    Ub = single.initial_state(_nonlinear_ic)
    multi.step(Ua, w.dt, 5)
    single.step(Ub, w.dt, 5)
    assert np.array_equal(Ua, Ub)
