"""Third-order P-ERK (P-ERK3) families as INPUT data (reading P3b).

The paper computes P-ERK3 coefficients offline (a nonlinear solve with a trust-region method from
random starting points, P:l.1085-1090) and the integrator consumes them.  Here the same offline step
is a deterministic, high-precision generator whose output -- the Butcher coefficients c, b and the
sub-diagonal a_{i,i-1} of every member -- is handed to BOTH the oracle and the CUDA library, exactly
like a level map.  Neither side trusts it: the oracle checks every family it is given against the
order conditions and the prescribed stability polynomial (tests/test_oracle_perk3.py), the library
checks internal consistency at perk_init.

Construction (paper: P:l.847-901 eqs. PERK_ThirdOrderShuOsher, Free_Timesteps; P:l.1067-1090
eq. PERK3_StabPnom and the third-order consistency condition):
  * c_i = (i-1)/(S-3), i = 1..S-2;  c_{S-1} = 1, c_S = 1/2 (Shu-Osher tail)
  * b_1 = b_{S-1} = 1/6, b_S = 4/6
  * member with E evaluations: unknowns x_i = a_{i,i-1}, i = S-E+3..S (all other a_{i,i-1} = 0),
    a_{i,1} = c_i - x_i; the z^{m+2} coefficient of its stability polynomial is
        b_S c_{S-m} prod_{j=S-m+1}^{S} x_j + b_{S-1} c_{S-1-m} prod_{j=S-m}^{S-1} x_j      (m >= 1)
    and must equal 1/6 (m = 1, the third-order condition b^T A c = 1/6) and alpha_{m+2}
    (m = 2..E-2).  Equation m determines x_{S-m} from x_{S-m+1..S} (x_{S-1} from x_S for m = 1), so
    the system collapses to one scalar equation g(x_S) = 0 (equation m = E-2, where the new unknown
    would be x_{S-E+2} = 0).
  * reading P3b: alpha_k = 1/k! (the Taylor rule of BASELINE cfg 1, as for P-ERK2); among the roots
    of g with all x_i in (0, c_i) and all a_{i,1} > 0 (the paper's positivity requirement) take the
    LARGEST x_S.  Roots are located on a grid and refined in 80-digit arithmetic (mpmath), including
    double roots (E = 4: g = -(8/3)(x_S - 1/8)^2).
This module imports nothing from oracle/ or paper_2403_05144_b200/.
"""
from __future__ import annotations

from fractions import Fraction as Fr
from functools import lru_cache
from math import factorial

import mpmath as mp

DPS = 80


def abscissae3(S: int) -> list:
    if S == 3:                                   # the Shu-Osher base itself: c = (0, 1, 1/2)
        return [Fr(0), Fr(1), Fr(1, 2)]
    return [Fr(i - 1, S - 3) for i in range(1, S - 1)] + [Fr(1), Fr(1, 2)]


def weights3(S: int) -> list:
    b = [Fr(0)] * S
    b[0], b[S - 2], b[S - 1] = Fr(1, 6), Fr(1, 6), Fr(4, 6)
    return b


def _chain(S, E, xS, c, b, alpha):
    """x_{S-E+3..S} (dict i -> x_i) from x_S by equations m = 1..E-3, and g(x_S) (equation E-2)."""
    x = {S: xS}
    if E == 3:
        return x, b[S - 1] * c[S - 2] * xS - mp.mpf(1) / 6          # m = 1 with x_{S-1} = 0
    x[S - 1] = (mp.mpf(1) / 6 - b[S - 1] * c[S - 2] * xS) / (b[S - 2] * c[S - 3])
    for m in range(2, E - 2):
        p_s = mp.mpf(1)
        for j in range(S - m + 1, S + 1):
            p_s *= x[j]
        p_s1 = mp.mpf(1)
        for j in range(S - m + 1, S):
            p_s1 *= x[j]
        # alpha_{m+2} = b_S c_{S-m} p_s + b_{S-1} c_{S-1-m} x_{S-m} p_s1
        x[S - m] = (alpha[m + 2] - b[S - 1] * c[S - m - 1] * p_s) / (b[S - 2] * c[S - m - 2] * p_s1)
    m = E - 2
    p_s = mp.mpf(1)
    for j in range(S - m + 1, S + 1):
        p_s *= x[j]
    return x, b[S - 1] * c[S - m - 1] * p_s - alpha[E]


def _admissible(x, c):
    return all(0 < v < c[i - 1] for i, v in x.items())


@lru_cache(maxsize=None)
def member3(S: int, E: int, alpha_rule: str = "taylor") -> dict:
    """x_i = a_{i,i-1} (i -> mpf) of the P-ERK3 member with E evaluations (reading P3b)."""
    assert 3 <= E <= S and S >= 3
    with mp.workdps(DPS):
        c = [mp.mpf(v.numerator) / v.denominator for v in abscissae3(S)]
        b = [mp.mpf(v.numerator) / v.denominator for v in weights3(S)]
        alpha = {k: mp.mpf(1) / factorial(k) for k in range(0, E + 1)}
        if alpha_rule != "taylor":
            raise ValueError(alpha_rule)
        if E == 3:
            x, _ = _chain(S, E, mp.mpf(1) / 4, c, b, alpha)
            return x
        g = lambda t: _chain(S, E, t, c, b, alpha)[1]
        hi = c[S - 1]
        n = 800
        grid = [hi * (k + 0.5) / n for k in range(n)]
        vals = [g(t) for t in grid]
        cands = []
        for k in range(n - 1):
            a, bb = vals[k], vals[k + 1]
            if a == 0:
                cands.append(grid[k])
            elif a * bb < 0:                                    # simple root: bisection
                lo_, hi_ = grid[k], grid[k + 1]
                for _ in range(280):                            # 2^-280 < 10^-80
                    mid = (lo_ + hi_) / 2
                    if g(lo_) * g(mid) <= 0:
                        hi_ = mid
                    else:
                        lo_ = mid
                cands.append((lo_ + hi_) / 2)
            if 0 < k < n - 1 and abs(vals[k]) <= abs(vals[k - 1]) and abs(vals[k]) <= abs(vals[k + 1]) \
                    and vals[k - 1] * vals[k + 1] > 0:
                # local extremum of g without a sign change: a double root if g vanishes there
                try:
                    t = mp.findroot(lambda s: mp.diff(g, s), grid[k])
                    if abs(g(t)) < mp.mpf(10) ** (-DPS // 2):
                        cands.append(t)
                except (ValueError, ZeroDivisionError):
                    pass
        good = []
        for t in cands:
            x, _ = _chain(S, E, t, c, b, alpha)
            if _admissible(x, c) and all(c[i - 1] - v > 0 for i, v in x.items()):
                good.append((t, x))
        if not good:
            raise ValueError(f"no admissible P-ERK3 member for S={S}, E={E}")
        return max(good, key=lambda p: p[0])[1]


def family3(S: int, E_list, alpha_rule: str = "taylor") -> dict:
    """A P-ERK3 family as doubles (c, b, a_sub[r][i-1] = a_{i,i-1}, a1 = c - a_sub) plus mpf values."""
    E_list = list(E_list)
    assert E_list == sorted(E_list) and E_list[0] >= 3 and E_list[-1] <= S
    c = abscissae3(S)
    b = weights3(S)
    asub_f, a1_f, asub_mp = [], [], []
    for E in E_list:
        x = member3(S, E, alpha_rule)
        row = [float(x.get(i, 0)) for i in range(1, S + 1)]
        asub_f.append(row)
        asub_mp.append(x)
        with mp.workdps(DPS):   # a_{i,1} = c_i - a_{i,i-1}, correctly rounded
            a1_f.append([float(mp.mpf(c[i].numerator) / c[i].denominator - x.get(i + 1, 0)) for i in range(S)])
    return dict(S=S, R=len(E_list), E=E_list, rule=alpha_rule, order=3, c=c, b=b,
                c_f=[float(v) for v in c], b_f=[float(v) for v in b], asub_f=asub_f, a1_f=a1_f, asub_mp=asub_mp)
