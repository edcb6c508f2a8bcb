"""Pins of the oracle's P-ERK2 tableau construction (oracle/tableau.py) against the paper.

* the printed compact table, PAPER.md l.535-561 (golden file)
* order conditions b^T 1 = 1, b^T c = 1/2 (l.227-247) and internal consistency (l.319-329)
* the closed form of the Taylor-rule family (derived)
* dt_max = 0.21875 for E = 8 on dx = 2/64 (l.564) via |P(dt lambda)| <= 1 on the Godunov spectrum
* brute force: one single-member step of the C oracle on a linear system equals
  sum_k alpha_k (dt L)^k U computed with explicit matrix powers.
"""
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

from oracle import oracle as O
from oracle import tableau as T

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load_compact():
    rows = []
    for line in open(os.path.join(GOLD, "perk2_s16_disk_compact.txt")):
        if line.startswith("#") or not line.strip():
            continue
        i, cnum, a8, a16 = line.split()
        rows.append((int(i), int(cnum), float(a8), float(a16)))
    return rows


def test_printed_compact_table_s16():
    fam = T.family(16, [8, 16], "disk")
    for i, cnum, a8, a16 in _load_compact():
        assert fam["c"][i - 1] == Fr(cnum, 30)
        for got, want in ((fam["asub_f"][0][i - 1], a8), (fam["asub_f"][1][i - 1], a16)):
            assert abs(got - want) <= 1e-14 * max(abs(want), 1e-300) or (want == 0 and got == 0)


@pytest.mark.parametrize("S,E", [(8, [4, 8]), (16, [4, 8, 16]), (28, [4, 6, 10, 16, 28]), (32, [4, 8, 16, 32]),
                                 (6, [4, 6])])
@pytest.mark.parametrize("rule", ["taylor", "disk"])
def test_order_conditions_and_consistency(S, E, rule):
    fam = T.family(S, E, rule)
    b, c = fam["b"], fam["c"]
    assert sum(b) == 1                                  # p = 1
    assert sum(bi * ci for bi, ci in zip(b, c)) == Fr(1, 2)   # p = 2
    for r in range(fam["R"]):
        for i in range(S):
            assert fam["a1"][r][i] + fam["asub"][r][i] == c[i]  # internal consistency, exact
        # member E evaluates {1} u {S-E+2..S}: a_{i,i-1} vanishes unless stage i-1 is evaluated
        for i in range(2, S + 1):
            if fam["asub"][r][i - 1] != 0:
                assert T.active(S, fam["E"][r], i - 1)


@pytest.mark.parametrize("S,E", [(8, [4, 8]), (16, [4, 8, 16]), (28, [4, 6, 10, 16, 28]), (32, [4, 8, 16, 32])])
def test_taylor_closed_form(S, E):
    """alpha_k = 1/k!  =>  a_{m,m-1} = (m-1)/((S-m+3)(m-2)) for m >= S-E+3, 0 otherwise."""
    fam = T.family(S, E, "taylor")
    for r, Er in enumerate(E):
        for m in range(1, S + 1):
            want = Fr(m - 1, (S - m + 3) * (m - 2)) if m >= S - Er + 3 else Fr(0)
            assert fam["asub"][r][m - 1] == want


def test_cfg1_values():
    fam = T.family(8, [4, 8], "taylor")
    assert fam["c"] == [Fr(i, 14) for i in range(8)]
    assert fam["asub"][1][2:] == [Fr(1, 4), Fr(3, 14), Fr(2, 9), Fr(1, 4), Fr(3, 10), Fr(7, 18)]
    assert fam["a1"][1][2:] == [Fr(-3, 28), Fr(0), Fr(4, 63), Fr(3, 28), Fr(9, 70), Fr(1, 9)]
    assert fam["asub"][0][:6] == [Fr(0)] * 6 and fam["asub"][0][6:] == [Fr(3, 10), Fr(7, 18)]


@pytest.mark.parametrize("rule", ["taylor", "disk"])
def test_stability_polynomial_roundtrip(rule):
    """eq. PERK2_StabPnom read off the constructed tableau gives back the prescribed alpha."""
    for S, E in ((16, [4, 8, 16]), (8, [4, 8])):
        fam = T.family(S, E, rule)
        for r, Er in enumerate(E):
            P = T.stability_poly(S, fam["c"], fam["asub"][r], Er)
            assert P == [fam["alpha"][r][k] for k in range(Er + 1)]


def test_disk_dt_max_e8():
    """dt = 0.21875 = 7/32 is the largest stable step of E = 8 on dx = 2/64."""
    al = T.alpha_disk(8)
    N, dx = 64, 2.0 / 64
    lam = (np.exp(-2j * np.pi * np.arange(N) / N) - 1.0) / dx
    P = lambda z: sum(float(al[k]) * z ** k for k in range(9))
    assert np.abs(P(0.21875 * lam)).max() <= 1 + 1e-12
    assert np.abs(P(0.21875 * 1.02 * lam)).max() > 1 + 1e-6


def _fv_matrix(dx, a=1.0):
    """L of eq. UpwindFullSystem: row i = (+a/dx_i at i-1, -a/dx_i at i), periodic."""
    n = len(dx)
    L = np.zeros((n, n))
    for i in range(n):
        L[i, i] = -a / dx[i]
        L[i, (i - 1) % n] = a / dx[i]
    return L


def test_fv_rhs_matches_paper_matrix():
    rng = np.random.default_rng(3)
    dx = rng.random(11) + 0.1
    L = _fv_matrix(dx)
    for _ in range(3):
        U = rng.standard_normal(11)
        assert np.allclose(O.fv_rhs(dx, U), L @ U, rtol=0, atol=1e-13 * np.abs(L).max() * np.abs(U).max())


@pytest.mark.parametrize("S,E,rule", [(8, 8, "taylor"), (16, 16, "disk"), (6, 6, "taylor")])
def test_bruteforce_stability_polynomial_fv(S, E, rule):
    """Single member, E = S: one step == sum_k alpha_k (dt L)^k U by explicit matrix powers."""
    fam = T.family(S, [E], rule)
    rng = np.random.default_rng(5)
    dx = 0.5 + rng.random(9)
    L = _fv_matrix(dx)
    dt = 0.3 * dx.min()
    U = rng.standard_normal(9)
    got = O.fv_step(dx, np.zeros(9, np.int32), fam, U, dt)
    al = fam["alpha"][0]
    want, Z = np.zeros(9), np.eye(9)
    for k in range(E + 1):
        want += float(al[k]) * (Z @ U)
        Z = (dt * L) @ Z
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


def test_bruteforce_stability_polynomial_dg():
    """Same pin through the DG oracle: 1D upwind DG advection, uniform 5 cells at max level, E = S = 8."""
    import workloads as W
    w = W.make(1, n_base=5)
    lm = np.ones_like(w.level_map)
    fam = T.family(8, [8], "taylor")
    m = O.OracleMesh(w.problem, lm, fam)
    nd = m.n * m.nv * m.npe
    L = np.zeros((nd, nd))
    for j in range(nd):
        e = np.zeros(nd)
        e[j] = 1.0
        L[:, j] = m.rhs(e.reshape(m.shape)).ravel()
    U = np.random.default_rng(1).standard_normal(nd)
    dt = 0.01
    got = U.copy().reshape(m.shape)
    m.step(got, dt)
    want, Z = np.zeros(nd), np.eye(nd)
    for k in range(9):
        want += float(fam["alpha"][0][k]) * (Z @ U)
        Z = (dt * L) @ Z
    assert np.abs(got.ravel() - want).max() <= 1e-12 * np.abs(want).max()
