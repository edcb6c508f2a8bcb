"""Workload generators for the five BASELINE.json configs (and reduced test sizes).

Everything here is *input*: a finest-grid level map (uint8, x fastest), an
analytic initial condition in conserved variables, a fixed dt and a step
count.  Readings of the configs follow SURVEY.md §8(c) P1-P10 and §8(d); they
are listed in DESIGN.md §3.  Nothing in this module depends on the DG
discretisation or on the P-ERK tableau.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import numpy as np

GAMMA = 1.4
N_POLY = 3  # DG polynomial degree fixed by BASELINE.json ("DGSEM N=3")

CONFIG_NAMES = {
    1: "cfg1_advection1d",
    2: "cfg2_euler1d",
    3: "cfg3_euler2d_static",
    4: "cfg4_euler2d_amr",
    5: "cfg5_ns2d",
}


@dataclasses.dataclass
class Workload:
    name: str
    problem: dict
    S: int
    E: list
    alpha_rule: str
    level_map: np.ndarray            # uint8, shape (nfx,) in 1D or (nfy, nfx) in 2D
    ic: Callable                     # ic(x) or ic(x, y) -> array (nv, *x.shape), conserved
    dt: float
    steps: int
    remesh_every: int = 0
    level_map_seq: Optional[Callable] = None   # k -> level map k (k >= 1), cfg 4
    seed: int = 0
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def nv(self) -> int:
        return self.problem["nv"]


# ----------------------------------------------------------------------------
# level-map utilities (valid finest-grid maps: every leaf is an aligned block)
# ----------------------------------------------------------------------------

def _blockmax(T: np.ndarray, s: int) -> np.ndarray:
    if T.ndim == 1:
        return T.reshape(-1, s).max(axis=1)
    ny, nx = T.shape
    return T.reshape(ny // s, s, nx // s, s).max(axis=(1, 3))


def _expand(B: np.ndarray, s: int) -> np.ndarray:
    if B.ndim == 1:
        return np.repeat(B, s)
    return np.repeat(np.repeat(B, s, axis=0), s, axis=1)


def leafify(T: np.ndarray, max_level: int) -> np.ndarray:
    """Smallest aligned-block tree whose leaves are at least as fine as T wants.

    A block of level l (edge 2^(max_level-l) finest cells) is a leaf iff no
    finest cell inside it asks for a level > l and no ancestor is a leaf.
    """
    T = np.asarray(T, dtype=np.int32)
    L = np.zeros(T.shape, dtype=np.int32)
    assigned = np.zeros(T.shape, dtype=bool)
    for lev in range(max_level + 1):
        s = 2 ** (max_level - lev)
        ok = _expand(_blockmax(T, s) <= lev, s)
        newly = ok & ~assigned
        L[newly] = lev
        assigned |= ok
    assert assigned.all()
    return L


def _shift(L: np.ndarray, d: int, axis: int, periodic: bool) -> np.ndarray:
    out = np.roll(L, d, axis=axis)
    if not periodic:
        idx = [slice(None)] * L.ndim
        idx[axis] = 0 if d > 0 else L.shape[axis] - 1
        out[tuple(idx)] = 0
    return out


def balance(L: np.ndarray, max_level: int, periodic=(True, True)) -> np.ndarray:
    """Enforce 2:1 balance across faces (corners not required), periodic wrap."""
    L = leafify(L, max_level)
    while True:
        T = L.copy()
        axes = [0] if L.ndim == 1 else [1, 0]  # x is the last axis in 2D
        for k, ax in enumerate(axes):
            per = periodic[k] if k < len(periodic) else True
            for d in (1, -1):
                T = np.maximum(T, _shift(L, d, ax, per) - 1)
        L2 = leafify(T, max_level)
        if np.array_equal(L2, L):
            return L.astype(np.uint8)
        L = L2


def _periodic_delta(a, b, period):
    d = np.abs(a - b) % period
    return np.minimum(d, period - d)


def _finest_centres_1d(lo, hi, nf):
    h = (hi - lo) / nf
    return lo + (np.arange(nf) + 0.5) * h


def _finest_centres_2d(lo, hi, nf):
    c = _finest_centres_1d(lo, hi, nf)
    X, Y = np.meshgrid(c, c, indexing="xy")  # shape (ny, nx), x fastest
    return X, Y


def _problem(dim, equation, volume, surface, n_base, max_level, lo, hi,
             periodic=(1, 1), gamma=GAMMA, prandtl=0.72, mu=0.0, adv=1.0,
             bc_state=(0.0, 0.0, 0.0, 0.0), max_cells=0):
    nv = {"advection": 1, "euler": 3 if dim == 1 else 4, "navier_stokes": 4}[equation]
    nb = (n_base, 1) if dim == 1 else (n_base, n_base)
    nf = nb[0] * 2 ** max_level
    return dict(dim=dim, equation=equation, volume=volume, surface=surface,
                n_base=nb, max_level=max_level, periodic=tuple(periodic),
                domain_lo=(lo, lo if dim == 2 else 0.0), domain_hi=(hi, hi if dim == 2 else 0.0),
                gamma=gamma, prandtl=prandtl, mu=mu, adv_velocity=adv,
                bc_state=tuple(bc_state), nv=nv, n_poly=N_POLY,
                max_cells=int(max_cells) if max_cells else (nf if dim == 1 else nf * nf),
                h_min=(hi - lo) / nf)


def _euler_speed_1d(U, gamma=GAMMA):
    rho, m, E = U
    v = m / rho
    p = (gamma - 1) * (E - 0.5 * rho * v * v)
    return np.abs(v) + np.sqrt(gamma * p / rho)


def _euler_speed_2d(U, gamma=GAMMA):
    rho, m1, m2, E = U
    v1, v2 = m1 / rho, m2 / rho
    p = (gamma - 1) * (E - 0.5 * rho * (v1 * v1 + v2 * v2))
    c = np.sqrt(gamma * p / rho)
    return np.maximum(np.abs(v1), np.abs(v2)) + c


def _cfl_dt(cfl, h_min, speed):
    """dt = CFL * h_min / ((N+1) * max wave speed)  (eqs. CFL_DG, TimestepConstraint)."""
    return float(cfl * h_min / ((N_POLY + 1) * speed))


# ----------------------------------------------------------------------------
# config 1: 1D linear advection, 2 levels, {4, 8}
# ----------------------------------------------------------------------------

def make_cfg1(seed=0, n_base=32, steps=200, cfl=0.2, refine_lo=-0.5, refine_hi=0.5):
    lo, hi, Lmax = -1.0, 1.0, 1
    nf = n_base * 2 ** Lmax
    xc = _finest_centres_1d(lo, hi, nf)
    T = ((xc > refine_lo) & (xc < refine_hi)).astype(np.int32)
    lmap = balance(T, Lmax, (True,))
    rng = np.random.default_rng(seed)
    A = rng.random(3)

    def ic(x, y=None):
        x = np.asarray(x, dtype=np.float64)
        u = sum(A[k] * np.sin((k + 1) * np.pi * x) for k in range(3))
        return u[None]

    prob = _problem(1, "advection", "weak", "upwind", n_base, Lmax, lo, hi, periodic=(1, 1))
    dt = _cfl_dt(cfl, prob["h_min"], 1.0)
    return Workload(CONFIG_NAMES[1], prob, 8, [4, 8], "taylor", lmap, ic, dt, steps,
                    seed=seed, meta=dict(amplitudes=A.tolist(), cfl=cfl))


# ----------------------------------------------------------------------------
# config 2: 1D Euler, 3 levels (two nested seeded windows), {4, 8, 16}
# ----------------------------------------------------------------------------

def make_cfg2(seed=0, n_base=256, steps=1000, cfl=0.2, w1=64, w2=16):
    lo, hi, Lmax = 0.0, 2.0, 2
    rng = np.random.default_rng(seed)
    o1 = int(rng.integers(0, n_base - w1 + 1))
    o2 = int(rng.integers(o1 + 1, o1 + w1 - w2))  # >= 1 base cell margin inside window 1
    T = np.zeros(n_base, dtype=np.int32)
    T[o1:o1 + w1] = 1
    T[o2:o2 + w2] = 2
    T = np.repeat(T, 2 ** Lmax)
    lmap = balance(T, Lmax, (True,))
    a = rng.normal(0.0, 0.01, 8)
    b = rng.normal(0.0, 0.01, 8)

    def rho0(x):
        eta = sum((a[k] * np.cos((k + 1) * np.pi * x) + b[k] * np.sin((k + 1) * np.pi * x)) / (k + 1)
                  for k in range(8))
        return 1.0 + 0.2 * np.sin(np.pi * x) + eta

    def ic(x, y=None):
        x = np.asarray(x, dtype=np.float64)
        rho = rho0(x)
        v = np.ones_like(x)
        p = np.ones_like(x)
        return np.stack([rho, rho * v, p / (GAMMA - 1) + 0.5 * rho * v * v])

    prob = _problem(1, "euler", "weak", "rusanov", n_base, Lmax, lo, hi, periodic=(1, 1))
    xs = np.linspace(lo, hi, 8 * n_base * 2 ** Lmax, endpoint=False)
    dt = _cfl_dt(cfl, prob["h_min"], _euler_speed_1d(ic(xs)).max())
    return Workload(CONFIG_NAMES[2], prob, 16, [4, 8, 16], "taylor", lmap, ic, dt, steps,
                    seed=seed, meta=dict(window1=(o1, w1), window2=(o2, w2), cfl=cfl))


# ----------------------------------------------------------------------------
# config 3: 2D Euler, static 3-level quadtree from seeded circles, {4, 8, 16}
# ----------------------------------------------------------------------------

def _circles_map(lo, hi, nf, Lmax, centres_per_level, radii):
    X, Y = _finest_centres_2d(lo, hi, nf)
    per = hi - lo
    T = np.zeros(X.shape, dtype=np.int32)
    for lev, (cs, r) in enumerate(zip(centres_per_level, radii), start=1):
        for (cx, cy) in cs:
            d2 = _periodic_delta(X, cx, per) ** 2 + _periodic_delta(Y, cy, per) ** 2
            T[d2 < r * r] = np.maximum(T[d2 < r * r], lev)
    return balance(T, Lmax, (True, True))


def _isentropic_vortices(centres, eps=5.0, per=10.0, background=(1.0, 1.0, 1.0, 1.0)):
    rho_inf, u_inf, v_inf, p_inf = background
    T_inf = p_inf / rho_inf

    def ic(x, y):
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        du = np.zeros_like(x)
        dv = np.zeros_like(x)
        dT = np.zeros_like(x)
        for (cx, cy) in centres:
            xb = (x - cx + per / 2) % per - per / 2   # nearest periodic image
            yb = (y - cy + per / 2) % per - per / 2
            r2 = xb * xb + yb * yb
            du += -eps / (2 * np.pi) * np.exp(0.5 * (1 - r2)) * yb
            dv += eps / (2 * np.pi) * np.exp(0.5 * (1 - r2)) * xb
            dT += -(GAMMA - 1) * eps * eps / (8 * GAMMA * np.pi * np.pi) * np.exp(1 - r2)
        Tt = T_inf + dT
        rho = rho_inf * (Tt / T_inf) ** (1.0 / (GAMMA - 1))
        p = rho * Tt
        u = u_inf + du
        v = v_inf + dv
        return np.stack([rho, rho * u, rho * v, p / (GAMMA - 1) + 0.5 * rho * (u * u + v * v)])

    return ic


def make_cfg3(seed=0, n_base=128, steps=500, cfl=0.2, radii=(2.2, 1.1), domain=10.0):
    lo, hi, Lmax = 0.0, domain, 2
    rng = np.random.default_rng(seed)
    centres = [rng.random((3, 2)) * domain for _ in range(Lmax)]
    nf = n_base * 2 ** Lmax
    lmap = _circles_map(lo, hi, nf, Lmax, centres, radii)
    vort = rng.random((3, 2)) * domain
    ic = _isentropic_vortices([tuple(c) for c in vort], per=domain)
    prob = _problem(2, "euler", "fluxdiff", "hll", n_base, Lmax, lo, hi, periodic=(1, 1))
    X, Y = _finest_centres_2d(lo, hi, nf)
    dt = _cfl_dt(cfl, prob["h_min"], _euler_speed_2d(ic(X, Y)).max())
    return Workload(CONFIG_NAMES[3], prob, 16, [4, 8, 16], "taylor", lmap, ic, dt, steps,
                    seed=seed, meta=dict(refine_centres=[c.tolist() for c in centres],
                                         vortex_centres=vort.tolist(), cfl=cfl))


# ----------------------------------------------------------------------------
# config 4: 2D Euler, dynamic AMR (moving bands), {4, 6, 10, 16, 28}
# ----------------------------------------------------------------------------

def _kh_bands_map(lo, hi, nf, Lmax, k, theta0, widths=(0.3, 0.15, 0.06, 0.015),
                  shift=0.01, dtheta=0.3):
    X, Y = _finest_centres_2d(lo, hi, nf)
    per = hi - lo
    T = np.zeros(X.shape, dtype=np.int32)
    s_k = shift * k
    th = theta0 + dtheta * k
    for sign in (+1.0, -1.0):
        yc = sign * 0.5 + s_k + 0.05 * np.sin(2 * np.pi * X + th)
        d = _periodic_delta(Y, yc, per)
        for lev, w in enumerate(widths[:Lmax], start=1):
            T[d < w] = np.maximum(T[d < w], lev)
    return balance(T, Lmax, (True, True))


def make_cfg4(seed=0, n_base=64, steps=2000, cfl=0.2, remesh_every=5, max_level=4,
              widths=(0.3, 0.15, 0.06, 0.015)):
    lo, hi, Lmax = -1.0, 1.0, max_level
    rng = np.random.default_rng(seed)
    theta0 = float(rng.random() * 2 * np.pi)
    A = float(0.05 + 0.05 * rng.random())
    phi = float(rng.random())
    nf = n_base * 2 ** Lmax

    def level_map_k(k):
        return _kh_bands_map(lo, hi, nf, Lmax, k, theta0, widths)

    def ic(x, y):
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        B = np.tanh(15 * y + 7.5) - np.tanh(15 * y - 7.5)
        rho = 0.5 + 0.25 * B
        u = 0.5 * (B - 1)
        v = A * np.sin(2 * np.pi * (x + phi))
        p = np.ones_like(x)
        return np.stack([rho, rho * u, rho * v, p / (GAMMA - 1) + 0.5 * rho * (u * u + v * v)])

    n_maps = steps // remesh_every + 1
    prob = _problem(2, "euler", "fluxdiff", "hll", n_base, Lmax, lo, hi, periodic=(1, 1),
                    max_cells=0)
    X, Y = _finest_centres_2d(lo, hi, nf)
    dt = _cfl_dt(cfl, prob["h_min"], _euler_speed_2d(ic(X, Y)).max())
    lmap0 = level_map_k(0)
    n0 = _count_leaves(lmap0, Lmax)
    prob["max_cells"] = int(2.2 * n0)
    return Workload(CONFIG_NAMES[4], prob, 28, [4, 6, 10, 16, 28], "taylor", lmap0, ic, dt, steps,
                    remesh_every=remesh_every, level_map_seq=level_map_k, seed=seed,
                    meta=dict(theta0=theta0, A=A, phi=phi, n_maps=n_maps, cfl=cfl,
                              # indicator-driven variant: enstrophy controller
                              # (P:l.1615-1622) replacing the seeded band sequence
                              amr=dict(indicator="enstrophy", variable="rho", base_level=0,
                                       med_level=min(2, Lmax), max_level=Lmax,
                                       med_threshold=1.0, max_threshold=15.0)))


# ----------------------------------------------------------------------------
# config 5: 2D Navier-Stokes (BR1), 4 levels, {4, 8, 16, 32}
# ----------------------------------------------------------------------------

def make_cfg5(seed=0, n_base=256, steps=200, cfl=0.2, radii=(1.3, 0.62, 0.3), mach=0.1, re=1600.0):
    lo, hi, Lmax = 0.0, 2 * np.pi, 3
    rng = np.random.default_rng(seed)
    centres = [rng.random((3, 2)) * (hi - lo) for _ in range(Lmax)]
    nf = n_base * 2 ** Lmax
    lmap = _circles_map(lo, hi, nf, Lmax, centres, radii)
    ph1, ph2 = rng.random(2) * 2 * np.pi

    def ic(x, y):
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        rho = np.ones_like(x)
        u = np.sin(x + ph1) * np.cos(y + ph2)
        v = -np.cos(x + ph1) * np.sin(y + ph2)
        p = 1.0 / (GAMMA * mach * mach) + 0.25 * (np.cos(2 * x) + np.cos(2 * y))
        return np.stack([rho, rho * u, rho * v, p / (GAMMA - 1) + 0.5 * rho * (u * u + v * v)])

    prob = _problem(2, "navier_stokes", "fluxdiff", "hll", n_base, Lmax, lo, hi, periodic=(1, 1),
                    mu=1.0 / re, prandtl=0.72)
    X, Y = _finest_centres_2d(lo, hi, nf)
    dt = _cfl_dt(cfl, prob["h_min"], _euler_speed_2d(ic(X, Y)).max())
    return Workload(CONFIG_NAMES[5], prob, 32, [4, 8, 16, 32], "taylor", lmap, ic, dt, steps,
                    seed=seed, meta=dict(refine_centres=[c.tolist() for c in centres],
                                         phases=[float(ph1), float(ph2)], cfl=cfl))


def _count_leaves(lmap, Lmax):
    lm = np.asarray(lmap, dtype=np.int64)
    d = lm.ndim
    return int(np.sum(1.0 / (2.0 ** (d * (Lmax - lm)))).round())


def make(cfg: int, seed: int = 0, **kw) -> Workload:
    return {1: make_cfg1, 2: make_cfg2, 3: make_cfg3, 4: make_cfg4, 5: make_cfg5}[cfg](seed=seed, **kw)


def count_leaves(w: Workload) -> int:
    return _count_leaves(w.level_map, w.problem["max_level"])


# ----------------------------------------------------------------------------
# shock-capturing inputs: a contact discontinuity on top of a workload's IC, so
# that the Hennemann-Gassner blending switches on in a band of elements (the paper's shock-capturing
# runs, P:l.1720-1731, start from discontinuous data)
# ----------------------------------------------------------------------------
SHOCK_CAPTURING = {"variable": "rho_p", "alpha_max": 0.5, "alpha_min": 0.001, "smooth": True}


def contact_band(ic, x0=0.35, width=0.12, factor=2.5, gamma=GAMMA):
    """2D IC wrapper: density x `factor` where |s - x0| < width, s = the x coordinate rescaled to
    [0, 1] over the nodes passed in; velocity and pressure unchanged"""
    def f(x, y):
        U = np.asarray(ic(x, y), np.float64)
        rho, vx, vy = U[0], U[1] / U[0], U[2] / U[0]
        p = (gamma - 1) * (U[3] - 0.5 * rho * (vx * vx + vy * vy))
        s = (x - x.min()) / (x.max() - x.min())
        rho = rho * np.where(np.abs(s - x0) < width, factor, 1.0)
        return np.stack([rho, rho * vx, rho * vy, p / (gamma - 1) + 0.5 * rho * (vx * vx + vy * vy)])
    return f
