"""Pins of the oracle's subcell shock capturing (perk_oracle.c section 9; DESIGN.md
A7-A9).  The paper runs its inviscid applications with the Hennemann-Gassner blending of the DGSEM
flux-differencing volume integral and a subcell finite-volume one (P:l.964, l.1729, l.1795-1799).
What the mathematics fixes:

* alpha = 1 everywhere: the scheme IS the first-order finite-volume method on the subcell grid
  (subcell widths w_i h / 2, the problem's surface flux between neighbouring nodes and across
  element faces) -- compared with an independent numpy FV written on the global node grid, so a
  wrong sign, a wrong weight, a transposed line or a dropped boundary term fails;
* alpha = 0 everywhere: bitwise the unblended flux-differencing operator;
* free-stream preservation for any alpha (constant states, mortars included);
* conservation (sum of the quadrature-weighted RHS vanishes, periodic, mortars, Euler and NS);
* the raw blending factor equals the pinned Hennemann-Gassner AMR indicator, and the smoothing
  equals max(alpha_e, alpha_n / 2) over face neighbours found by a geometric brute-force search;
* the restricted (per-member list) P-ERK step equals the reference-mode step bitwise.
"""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from oracle import tableau as T

G = 1.4
WQ = np.array([1.0, 5.0, 5.0, 1.0]) / 6.0
FAM1 = T.family(4, [4], "taylor")
FAM2 = T.family(6, [3, 6], "taylor")


def _prob(nb, L, sc=None, eq="euler", surface="hll"):
    p = W.configs._problem(2, eq, "fluxdiff", surface, nb, L, 0.0, 1.0, periodic=(1, 1))
    if eq == "navier_stokes":
        p["mu"], p["prandtl"] = 1e-3, 0.72
    if sc is not None:
        p["shock_capturing"] = sc
    return p


def _mortar_map(nb=2, L=1):
    lm = np.zeros((nb << L, nb << L), np.uint8)
    lm[0:2, 0:2] = 1
    return lm


def _three_level_map():
    """levels 0, 1, 2 on an 8 x 8 finest grid (2 x 2 base cells, L = 2), 2:1 balanced, periodic"""
    lm = np.ones((8, 8), np.uint8)
    lm[0:2, 0:2] = 2
    lm[4:8, 4:8] = 0
    return lm


def _state(m, seed=0, amp=0.1, jump=False):
    """smooth positive random state; jump=True adds a density / pressure discontinuity"""
    xy = m.node_coords()
    x, y = xy[:, 0, :], xy[:, 1, :]
    rng = np.random.default_rng(seed)
    k = rng.uniform(0.5, 2.0, 6)
    rho = 1.0 + amp * np.sin(2 * np.pi * (x + k[0] * y)) + amp * 0.5 * np.cos(2 * np.pi * k[1] * x)
    vx = 0.3 + amp * np.sin(2 * np.pi * (k[2] * x - y))
    vy = -0.2 + amp * np.cos(2 * np.pi * (x + k[3] * y))
    p = 1.0 + amp * np.cos(2 * np.pi * (k[4] * x + y))
    if jump:
        rho = rho + 0.8 * (np.abs(x - 0.5) < 0.2)
        p = p + 1.5 * (np.abs(y - 0.45) < 0.15)
    U = np.stack([rho, rho * vx, rho * vy, p / (G - 1) + 0.5 * rho * (vx * vx + vy * vy)], 1)
    return np.ascontiguousarray(U)


def _hll(uL, uR, d):
    """HLL with Davis wave speeds, arrays (4, ...) of conserved states, direction d (independent)"""
    def prim(u):
        r = u[0]
        v = u[1 + d] / r
        p = (G - 1) * (u[3] - 0.5 * (u[1] ** 2 + u[2] ** 2) / r)
        f = np.stack([u[1 + d], u[1] * v, u[2] * v, (u[3] + p) * v])
        f[1 + d] += p
        return f, v, np.sqrt(G * p / r)
    fL, vL, cL = prim(uL)
    fR, vR, cR = prim(uR)
    sL = np.minimum(vL - cL, vR - cR)
    sR = np.maximum(vL + cL, vR + cR)
    mid = (sR * fL - sL * fR + sL * sR * (uR - uL)) / (sR - sL)
    return np.where(sL >= 0, fL, np.where(sR <= 0, fR, mid))


def test_alpha_one_is_global_subcell_fv():
    nb = 3
    m = O.OracleMesh(_prob(nb, 0, {"alpha_fixed": 1.0}), np.zeros((nb, nb), np.uint8), FAM1)
    U = _state(m, seed=3, amp=0.2)
    dU = m.rhs(U)
    lv = m.leaves()
    h = 1.0 / nb
    # global node grid: gx = 4 * column + i, gy = 4 * row + j
    Gs = np.zeros((4, 4 * nb, 4 * nb))
    for e in range(m.n):
        cx, cy = lv["fx"][e], lv["fy"][e]
        Gs[:, 4 * cy:4 * cy + 4, 4 * cx:4 * cx + 4] = U[e].reshape(4, 4, 4)
    width = np.tile(WQ * h / 2, nb)
    Fx = _hll(Gs, np.roll(Gs, -1, axis=2), 0)            # flux between gx and gx + 1 (periodic)
    Fy = _hll(Gs, np.roll(Gs, -1, axis=1), 1)
    ref = -(Fx - np.roll(Fx, 1, axis=2)) / width[None, None, :] - (Fy - np.roll(Fy, 1, axis=1)) / width[None, :, None]
    got = np.zeros_like(Gs)
    for e in range(m.n):
        cx, cy = lv["fx"][e], lv["fy"][e]
        got[:, 4 * cy:4 * cy + 4, 4 * cx:4 * cx + 4] = dU[e].reshape(4, 4, 4)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))


def test_alpha_one_rusanov_surface_flux():
    """the subcell flux is the problem's surface flux: with Rusanov, alpha = 1 is Rusanov FV
    (its interior subcell fluxes cannot be HLL: the results differ)"""
    nb = 2
    lm = np.zeros((nb, nb), np.uint8)
    a = O.OracleMesh(_prob(nb, 0, {"alpha_fixed": 1.0}, surface="rusanov"), lm, FAM1)
    b = O.OracleMesh(_prob(nb, 0, {"alpha_fixed": 1.0}), lm, FAM1)
    U = _state(a, seed=4, amp=0.2)
    assert np.max(np.abs(a.rhs(U) - b.rhs(U))) > 1e-6


@pytest.mark.parametrize("eq", ["euler", "navier_stokes"])
def test_alpha_zero_is_bitwise_unblended(eq):
    lm = _mortar_map()
    a = O.OracleMesh(_prob(2, 1, {"alpha_fixed": 0.0}, eq=eq), lm, FAM1)
    b = O.OracleMesh(_prob(2, 1, None, eq=eq), lm, FAM1)
    U = _state(a, seed=1, amp=0.2, jump=True)
    assert np.array_equal(a.rhs(U), b.rhs(U))


@pytest.mark.parametrize("alpha", [0.3, 1.0, None])
def test_free_stream(alpha):
    lm = _mortar_map()
    m = O.OracleMesh(_prob(2, 1, {"alpha_fixed": alpha}), lm, FAM1)
    U = np.zeros(m.shape)
    U[:, 0], U[:, 1], U[:, 2], U[:, 3] = 1.2, 1.2 * 0.4, -1.2 * 0.3, 2.0 / (G - 1) + 0.5 * 1.2 * 0.25
    assert np.max(np.abs(m.rhs(U))) < 1e-12


@pytest.mark.parametrize("eq", ["euler", "navier_stokes"])
def test_conservation_with_mortars(eq):
    lm = _three_level_map()
    m = O.OracleMesh(_prob(2, 2, {"variable": "rho_p", "alpha_max": 1.0}, eq=eq), lm, FAM1)
    U = _state(m, seed=2, amp=0.2, jump=True)
    raw, sm = m.sc_alpha(U)
    assert raw.max() > 0.1 and (raw == 0).any() and sm.max() == 1.0   # blended and pure-DG elements
    dU = m.rhs(U)
    lev = m.leaves()["level"]
    h = 1.0 / (2 << 2) * (2.0 ** (2 - lev.astype(float)))
    wq = np.outer(WQ, WQ).ravel()
    tot = np.einsum("e,evq,q->v", (h / 2) ** 2, dU, wq)
    scale = np.einsum("e,evq,q->v", (h / 2) ** 2, np.abs(dU), wq)
    assert np.all(np.abs(tot) <= 1e-13 * scale)


def _neighbours(lv, nf):
    """face neighbours of every leaf by geometry (periodic square of nf finest cells)"""
    n = len(lv["fx"])
    L = int(lv["level"].max())
    s = [(1 << (L - int(l))) for l in lv["level"]]
    box = [(int(lv["fx"][e]), int(lv["fy"][e]), s[e]) for e in range(n)]
    nb = [set() for _ in range(n)]
    for a in range(n):
        xa, ya, sa = box[a]
        for b in range(n):
            if a == b:
                continue
            xb, yb, sb = box[b]
            for dx in (-nf, 0, nf):
                for dy in (-nf, 0, nf):
                    x0, y0 = xb + dx, yb + dy
                    touch_x = (x0 == xa + sa or x0 + sb == xa) and min(ya + sa, y0 + sb) - max(ya, y0) > 0
                    touch_y = (y0 == ya + sa or y0 + sb == ya) and min(xa + sa, x0 + sb) - max(xa, x0) > 0
                    if touch_x or touch_y:
                        nb[a].add(b)
    return nb


def test_smoothing_matches_brute_force_neighbours():
    """4 x 4 base cells, levels 0-2 (64 leaves, interfaces AND mortars between blended and unblended
    elements, intermediate alpha values)"""
    L = 2
    lm = np.ones((16, 16), np.uint8)
    lm[0:4, 0:4] = 2
    lm[8:16, 8:16] = 0
    p = W.configs._problem(2, "euler", "fluxdiff", "hll", 4, L, 0.0, 1.0, periodic=(1, 1))
    p["shock_capturing"] = {"variable": "rho", "alpha_max": 0.8, "alpha_min": 0.001}
    m = O.OracleMesh(p, lm, FAM1)
    U = _state(m, seed=4, amp=0.2, jump=True)
    raw, sm = m.sc_alpha(U)
    ind = m.amr_indicator(U, {"indicator": "hennemann_gassner", "variable": "rho", "base_level": 0,
                              "med_level": 0, "max_level": L, "med_threshold": 0.1, "max_threshold": 0.5,
                              "alpha_max": 0.8, "alpha_min": 0.001})
    assert np.array_equal(raw, ind)
    assert 0 < np.count_nonzero(raw) < m.n and ((raw > 0.01) & (raw < 0.79)).any()
    f, _ = m.faces("interfaces")
    assert sum(1 for a, b, o in f if raw[a] != raw[b]) > 10      # interfaces between differing alphas
    assert m.face_counts()["mortars"] > 0
    nbrs = _neighbours(m.leaves(), 4 << L)
    exp = np.array([max([raw[e]] + [0.5 * raw[b] for b in nbrs[e]]) for e in range(m.n)])
    assert np.array_equal(sm, exp)
    assert not np.array_equal(sm, raw)                  # the smoothing changed something
    p2 = dict(p, shock_capturing={"variable": "rho", "alpha_max": 0.8, "smooth": False})
    raw2, sm2 = O.OracleMesh(p2, lm, FAM1).sc_alpha(U)
    assert np.array_equal(sm2, raw2) and np.array_equal(raw2, raw)


def test_restricted_step_equals_reference():
    L = 2
    lm = _three_level_map()
    m = O.OracleMesh(_prob(2, L, {"variable": "rho_p"}), lm, FAM2)
    U0 = _state(m, seed=6, amp=0.2, jump=True)
    a, b = U0.copy(), U0.copy()
    m.step(a, 2e-3, 2, mode=1)
    m.step(b, 2e-3, 2, mode=0)
    assert np.array_equal(a, b)
    assert np.max(np.abs(a - U0)) > 1e-4


def test_invalid_parameters():
    with pytest.raises(ValueError):
        O.OracleMesh(_prob(2, 0, {"alpha_max": 1.5}), np.zeros((2, 2), np.uint8), FAM1)
    p1 = W.configs._problem(1, "euler", "weak", "rusanov", 4, 0, 0.0, 1.0)
    p1["shock_capturing"] = {}
    with pytest.raises(ValueError):
        O.OracleMesh(p1, np.zeros(4, np.uint8), FAM1)


def test_contact_band_input():
    """the shock-capturing input (workloads.configs.contact_band): density x 2.5 inside the band,
    velocity and pressure of the base IC unchanged everywhere"""
    w = W.make(3, n_base=8)
    m = O.OracleMesh(w.problem, w.level_map, FAM1)
    U0 = m.initial_state(w.ic)
    U1 = m.initial_state(W.configs.contact_band(w.ic))
    def prim(U):
        r = U[:, 0]
        vx, vy = U[:, 1] / r, U[:, 2] / r
        return r, vx, vy, (G - 1) * (U[:, 3] - 0.5 * r * (vx * vx + vy * vy))
    r0, vx0, vy0, p0 = prim(U0)
    r1, vx1, vy1, p1 = prim(U1)
    ratio = r1 / r0
    assert np.allclose(vx1, vx0, rtol=1e-13, atol=1e-13) and np.allclose(vy1, vy0, rtol=1e-13, atol=1e-13)
    assert np.allclose(p1, p0, rtol=1e-12)
    inside = np.isclose(ratio, 2.5, rtol=1e-14)
    assert np.all(inside | np.isclose(ratio, 1.0, rtol=1e-14))
    x = m.node_coords()[:, 0, :]
    s = (x - x.min()) / (x.max() - x.min())
    assert np.array_equal(inside, np.abs(s - 0.35) < 0.12)
