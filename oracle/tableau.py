"""ORACLE -- TEST INFRASTRUCTURE ONLY.  P-ERK2 tableaux in exact rational arithmetic.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this module.  The CUDA path builds its own tableau (C, double) and
never imports anything under oracle/.

Paper:
  * standard pattern, shared c and b = e_S, a_{i,1} = c_i - a_{i,i-1}
    (l.407-436, eq. PERK_ButcherTableauClassic; l.319-329 eq. InternalConsistency; l.533)
  * c_i = (i-1) / (2 (S-1))  (l.416-421 for S = 6, l.542-559 for S = 16; BASELINE.json cfg 1)
  * stability polynomial P_{2;E}(z) = 1 + z + z^2/2 + sum_{k=3}^{E} alpha_k z^k with
    alpha_k = c_{S-k+2} prod_{i=S-k+3}^{S} a_i  (l.1048-1056, eq. PERK2_StabPnom, exponent read
    as z^E)
  * recursion a_{S-i} = alpha_{3+i} / (c_{S-i-1} prod_{j<i} a_{S-j}), i = 0..E-3
    (l.1058-1064, eq. PERKCoeffsConstruction; range read as E-3)
Polynomial rules:
  * "taylor": alpha_k = 1/k!  (BASELINE.json cfg 1; used for all configs)
  * "disk":   P_E(z) = 1/E + ((E-1)/E) (1 + z/(E-1))^E, the second-order optimum for the
              circular Godunov spectrum (l.513-520); reproduces the table at l.535-561.
Parity: pinned by tests/test_oracle_tableau.py (printed table, closed forms, brute force).
"""
from __future__ import annotations

from fractions import Fraction as Fr
from math import comb, factorial


def abscissae(S: int) -> list:
    """c_1..c_S (index 0..S-1)."""
    return [Fr(i - 1, 2 * (S - 1)) for i in range(1, S + 1)]


def alpha_taylor(E: int) -> dict:
    return {k: Fr(1, factorial(k)) for k in range(0, E + 1)}


def alpha_disk(E: int) -> dict:
    # coefficients of 1/E + ((E-1)/E)(1 + z/(E-1))^E
    out = {}
    for k in range(0, E + 1):
        a = Fr(E - 1, E) * comb(E, k) * Fr(1, (E - 1) ** k) if E > 1 else Fr(1 if k <= 1 else 0)
        if k == 0:
            a += Fr(1, E)
        out[k] = a
    return out


def member_a_sub(S: int, E: int, alpha: dict) -> list:
    """a_{i,i-1} for i = 1..S (index i-1) of the member with E evaluations (eq. PERKCoeffsConstruction)."""
    c = abscissae(S)
    a = {}
    for i in range(0, E - 2):             # i = 0..E-3
        prod = Fr(1)
        for j in range(0, i):
            prod *= a[S - j]
        a[S - i] = alpha[3 + i] / (c[S - i - 1 - 1] * prod)   # c_{S-i-1} is index S-i-2
    return [a.get(i, Fr(0)) for i in range(1, S + 1)]


def family(S: int, E_list, rule: str = "taylor") -> dict:
    """The P-ERK2 family {E_1 < ... < E_R = S}; exact Fractions plus rounded doubles."""
    E_list = list(E_list)
    assert E_list == sorted(E_list) and len(set(E_list)) == len(E_list)
    assert E_list[-1] <= S and E_list[0] >= 2
    c = abscissae(S)
    rules = {"taylor": alpha_taylor, "disk": alpha_disk}
    asub, a1, alphas = [], [], []
    for E in E_list:
        al = rules[rule](E)
        s = member_a_sub(S, E, al)
        asub.append(s)
        a1.append([c[i] - s[i] for i in range(S)])
        alphas.append(al)
    b = [Fr(0)] * (S - 1) + [Fr(1)]
    return dict(S=S, R=len(E_list), E=E_list, rule=rule, c=c, b=b, asub=asub, a1=a1, alpha=alphas,
                c_f=[float(x) for x in c],
                asub_f=[[float(x) for x in row] for row in asub],
                a1_f=[[float(x) for x in row] for row in a1])


def stability_poly(S: int, c: list, a_sub_member: list, E: int) -> list:
    """Monomial coefficients of P_{2;E} read off eq. PERK2_StabPnom from the tableau."""
    out = [Fr(1), Fr(1), Fr(1, 2)]
    for k in range(3, E + 1):
        prod = Fr(1)
        for i in range(S - k + 3, S + 1):
            prod *= a_sub_member[i - 1]
        out.append(c[S - k + 2 - 1] * prod)
    return out


def active(S: int, E: int, i: int) -> bool:
    """Member E evaluates stage i (1-based) iff i == 1 or i >= S - E + 2 (eq. PERK_ButcherTableauClassic)."""
    return i == 1 or i >= S - E + 2
