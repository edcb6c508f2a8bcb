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
Stage patterns and weights (F1-F3):
  * "standard" {1} u {S-E+2..S} (l.407-436); "early" shared evaluations {1..E-1} u {S}
    (l.683-700: S = 6, E = 4 -> {1, 2, 3, 6}); "alternating" {1} u {S - floor((E-1-k)(S-1)/(E-1) + 1/2),
    k = 1..E-1} (l.655-675: S = 6, E = 4 -> {1, 3, 4, 6}); or an explicit stage set.  Stage i's row
    has a_{i,1} and a_{i,p(i)}, p(i) = the member's previous evaluated stage > 1; the first evaluated
    stage after 1 has only a_{i,1} = c_i.
  * weights b_S = 1/(2 c_S), b_1 = 1 - b_S with c_i = c_S (i-1)/(S-1) (l.439-442: c_S = 1/2 the
    standard midpoint choice, 1 Heun, 2/3 Ralston).
  * along a member's chain s_1 < ... < s_{E-1} = S of evaluated stages after 1 the stability
    polynomial is 1 + z + sum_{j>=2} alpha_{j+1} z^{j+1} with alpha_{j+1} = b_S c_{s_{E-j}} prod_{m=E-j+1}^{E-1} a_m
    (a_m the row coefficient of stage s_m), the pattern-independent generalisation of eq. PERK2_StabPnom,
    so a_{E-1-i} = alpha_{3+i} / (b_S c_{s_{E-2-i}} prod_{m<i} a_{E-1-m}), i = 0..E-3.
Parity: pinned by tests/test_oracle_tableau.py (printed table, closed forms, brute force) and
tests/test_oracle_patterns.py (printed pattern tableaux, matrix powers, Heun / Ralston at S = 2).
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


def pattern_stages(S: int, E: int, pattern="standard") -> list:
    """Evaluated stages (1-based, ascending) of a member with E evaluations."""
    if pattern == "standard":
        st = [1] + list(range(S - E + 2, S + 1))
    elif pattern == "early":
        st = list(range(1, E)) + [S]
    elif pattern == "alternating":
        st = [1] + [S - ((E - 1 - k) * (S - 1) * 2 + (E - 1)) // (2 * (E - 1)) for k in range(1, E)]
    else:
        st = sorted(int(i) for i in pattern)
    assert len(st) == E and len(set(st)) == E and st[0] == 1 and st[-1] == S, (S, E, pattern, st)
    return st


def member_chain_a_sub(S: int, E: int, alpha: dict, stages: list, c: list, bS=Fr(1)) -> list:
    """row coefficients a_{i,p(i)} (index i-1) along the member's chain of evaluated stages"""
    s = stages[1:]                                   # s_1 .. s_{E-1}, s_{E-1} = S
    a = {}                                           # chain position k -> a_k (k = 2..E-1)
    for i in range(0, E - 2):
        k = E - 1 - i
        prod = Fr(1)
        for m in range(k + 1, E):
            prod *= a[m]
        a[k] = alpha[3 + i] / (bS * c[s[k - 2] - 1] * prod)     # c_{s_{k-1}}
    out = [Fr(0)] * S
    for k, v in a.items():
        out[s[k - 1] - 1] = v
    return out


def family(S: int, E_list, rule: str = "taylor", pattern="standard", c_S=Fr(1, 2)) -> dict:
    """The P-ERK2 family {E_1 < ... < E_R = S}; exact Fractions plus rounded doubles.
    pattern: one pattern for every member, or a list with one per member (name or stage set)."""
    E_list = list(E_list)
    assert E_list == sorted(E_list) and len(set(E_list)) == len(E_list)
    assert E_list[-1] <= S and E_list[0] >= 2
    c_S = Fr(c_S)
    c = abscissae(S) if c_S == Fr(1, 2) else [c_S * Fr(i - 1, S - 1) for i in range(1, S + 1)]
    bS = 1 / (2 * c_S)
    rules = {"taylor": alpha_taylor, "disk": alpha_disk}
    pats = pattern if isinstance(pattern, (list, tuple)) and len(pattern) == len(E_list) and \
        not all(isinstance(x, int) for x in pattern) else [pattern] * len(E_list)
    asub, a1, alphas, stages = [], [], [], []
    for E, pat in zip(E_list, pats):
        al = rules[rule](E)
        st = pattern_stages(S, E, pat)
        s = member_a_sub(S, E, al) if (st == pattern_stages(S, E) and bS == 1) else \
            member_chain_a_sub(S, E, al, st, c, bS)
        asub.append(s)
        a1.append([c[i] - s[i] for i in range(S)])
        alphas.append(al)
        stages.append(st)
    b = [Fr(0)] * S
    b[0] += 1 - bS
    b[S - 1] += bS
    standard = all(st == pattern_stages(S, E) for st, E in zip(stages, E_list))
    return dict(S=S, R=len(E_list), E=E_list, rule=rule, c=c, b=b, asub=asub, a1=a1, alpha=alphas,
                stages=stages, pattern=pattern,
                active_mask=None if standard else [sum(1 << (i - 1) for i in st) for st in stages],
                c_f=[float(x) for x in c], b_f=[float(x) for x in b],
                asub_f=[[float(x) for x in row] for row in asub],
                a1_f=[[float(x) for x in row] for row in a1])


def butcher(fam: dict, r: int) -> list:
    """dense S x S Butcher matrix A^(r) of member r (exact), rows i = 1..S"""
    S = fam["S"]
    A = [[Fr(0)] * S for _ in range(S)]
    st = fam["stages"][r]
    for i in range(2, S + 1):
        prev = [j for j in st if 1 < j < i]
        a = fam["asub"][r][i - 1]
        if a != 0:
            assert i in st and prev, (r, i)
            A[i - 1][prev[-1] - 1] = a
        A[i - 1][0] = fam["c"][i - 1] - a
    return A


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
