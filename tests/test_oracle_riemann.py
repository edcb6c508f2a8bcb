"""Pins of the oracle's Euler surface fluxes (Rusanov / local Lax-Friedrichs and HLL with Davis
wave speeds) by the mathematics of their linearisation, independent of the flux formulas.

PAPER.md l.1545 names the Rusanov / LLF surface flux (BASELINE.json configs[1], cfg 2); HLL is the
cfg 3-5 surface flux.  Neither the paper nor a closed-form solution fixes the
wave speed these fluxes use, and the cfg-2 contact invariant is blind to it (with v and p constant
every flux component is affine in the mass flux).  What pins it:

About a constant state u0 = (rho0, v0, p0) the DG operator of the Euler equations linearises to
J = dF/dU.  The flux Jacobian A of the Euler equations at u0 (computed here by differencing the
PDE's flux function, not the oracle's) has eigenvalues a_k = v0 - c, v0, v0 + c with the textbook
sound speed c = sqrt(gamma p0 / rho0), and the same eigenvector matrix R at every node, so in
characteristic variables w = R^-1 u the linearised operator decouples into scalar DG operators
L(a, d): speed a, surface flux a {{w}} - (d / 2) [[w]] (central part plus dissipation d).  Both
parts are linear, so L(a, d) = a C + d D with C = (L_+ - L_-)/2 and D = (L_+ + L_-)/2, where L_+
and L_- are the oracle's own upwind linear-advection operators for speeds +1 and -1 (pinned by
the cfg-1 exact-solution tests).  The fluxes' dissipation coefficients follow from their
definitions at a constant state:
  * Rusanov: d = lambda = |v0| + c for every wave (one wave speed bound for all),
  * HLL (s_L = v0 - c, s_R = v0 + c): d_k = (a_k (s_R + s_L) - 2 s_L s_R) / (s_R - s_L), which is
    |a_k| (upwind) for the two acoustic waves and c for the entropy wave.
A wrong sound speed, a wave speed without the sound speed, or a wrong HLL combination changes the
block diagonal (the mutation check in DESIGN.md §9 lists the mutants this catches).  The 2D
version takes perturbations that are constant in y on a uniform mesh: the operator maps that
subspace to itself and acts there as the 1D one with the x-flux Jacobian (eigenvalues v1 - c, v1,
v1, v1 + c).
"""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from oracle import tableau as T

GAMMA = 1.4


def _euler_flux_1d(U):
    rho, m, E = U
    v = m / rho
    p = (GAMMA - 1) * (E - 0.5 * rho * v * v)
    return np.array([m, m * v + p, (E + p) * v])


def _euler_flux_x_2d(U):
    rho, m1, m2, E = U
    v1, v2 = m1 / rho, m2 / rho
    p = (GAMMA - 1) * (E - 0.5 * rho * (v1 * v1 + v2 * v2))
    return np.array([m1, m1 * v1 + p, m2 * v1, (E + p) * v1])


def _fd_jacobian(f, u0, eps=1e-6):
    n = len(u0)
    J = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = eps
        J[:, j] = (f(u0 + e) - f(u0 - e)) / (2 * eps)
    return J


def _char_basis(A, c, v0):
    """Eigenvectors of the flux Jacobian for the textbook eigenvalues v0 - c, v0 (once in 1D,
    twice in 2D), v0 + c: for each, the null space of A - mu I (smallest right-singular vectors,
    whose singular values must vanish), so the repeated eigenvalue gets a well-conditioned basis."""
    nv = A.shape[0]
    lam = np.array([v0 - c] + [v0] * (nv - 2) + [v0 + c])
    cols = []
    for mu, mult in ((v0 - c, 1), (v0, nv - 2), (v0 + c, 1)):
        _, sv, Vt = np.linalg.svd(A - mu * np.eye(nv))
        assert sv[-mult:].max() < 1e-7 * np.abs(A).max(), (mu, sv)
        cols += [Vt[-1 - k] for k in range(mult)]
    R = np.array(cols).T
    assert np.linalg.cond(R) < 1e3
    return lam, R, np.linalg.inv(R)


def _mesh(dim, equation, surface, n_base, adv=1.0):
    prob = W.configs._problem(dim, equation, "weak" if dim == 1 else "fluxdiff", surface, n_base, 0,
                              0.0, 2.0, adv=adv)
    lm = np.zeros(n_base if dim == 1 else (n_base, n_base), dtype=np.uint8)
    return O.OracleMesh(prob, lm, T.family(4, [4], "taylor"))


def _advection_parts(n_base):
    """C and D of the scalar DG operator (section docstring) from the oracle's upwind advection."""
    ops = []
    for a in (1.0, -1.0):
        m = _mesh(1, "advection", "upwind", n_base, adv=a)
        nd = m.n * m.npe
        L = np.zeros((nd, nd))
        for j in range(nd):
            e = np.zeros(nd)
            e[j] = 1.0
            L[:, j] = m.rhs(e.reshape(m.shape)).ravel()
        ops.append(L)
    Lp, Lm = ops
    return 0.5 * (Lp - Lm), 0.5 * (Lp + Lm)


def _dissipation(surface, lam, v0, c):
    if surface == "rusanov":
        return np.full(len(lam), abs(v0) + c)
    sL, sR = v0 - c, v0 + c
    return (lam * (sR + sL) - 2 * sL * sR) / (sR - sL)


def _ddir(m, U0, d, eps=2e-6):
    """Directional derivative of the oracle's RHS at U0 along d.  The wave-speed bounds contain
    |v| and max(left, right), which are not differentiable at a constant state; they multiply a
    jump that vanishes there, so the central difference carries an O(eps) term, removed by one
    Richardson step."""
    def cd(h):
        return (m.rhs(U0 + h * d) - m.rhs(U0 - h * d)) / (2 * h)
    return 2 * cd(eps / 2) - cd(eps)


def _linearised_1d(m, U0):
    """J[(e,i) x (e',i')] blocks [v, v'] of the oracle's RHS about the constant state U0."""
    n, nv, npe = m.shape
    J = np.zeros((n, nv, npe, n, nv, npe))
    for e in range(n):
        for v in range(nv):
            for i in range(npe):
                d = np.zeros(m.shape)
                d[e, v, i] = 1.0
                J[:, :, :, e, v, i] = _ddir(m, U0, d)
    return J


@pytest.mark.parametrize("surface", ["rusanov", "hll"])
@pytest.mark.parametrize("state", [(1.0, 0.0, 1.0), (1.3, 0.3, 0.8), (0.7, -0.45, 1.6)])
def test_euler1d_linearised_flux_decouples(surface, state):
    rho0, v0, p0 = state
    n_base = 6
    c = np.sqrt(GAMMA * p0 / rho0)
    u0 = np.array([rho0, rho0 * v0, p0 / (GAMMA - 1) + 0.5 * rho0 * v0 * v0])
    lam, R, Ri = _char_basis(_fd_jacobian(_euler_flux_1d, u0), c, v0)
    d = _dissipation(surface, lam, v0, c)
    if surface == "hll":   # the closed form reduces to upwind for the acoustic waves
        assert abs(d[0] - abs(v0 - c)) < 1e-9 and abs(d[2] - abs(v0 + c)) < 1e-9
        assert abs(d[1] - c) < 1e-9
    Cm, Dm = _advection_parts(n_base)
    m = _mesh(1, "euler", surface, n_base)
    U0 = np.broadcast_to(u0[None, :, None], m.shape).copy()
    J = _linearised_1d(m, U0)
    n, nv, npe = m.shape
    Jc = np.einsum("kv,evifuj,ul->ekiflj", Ri, J, R)
    scale = np.abs(Jc).max()
    for k in range(nv):
        for l in range(nv):
            blk = Jc[:, k, :, :, l, :].reshape(n * npe, n * npe)
            expect = lam[k] * Cm + d[k] * Dm if k == l else np.zeros_like(blk)
            assert np.abs(blk - expect).max() < 1e-8 * scale, (k, l, np.abs(blk - expect).max())


@pytest.mark.parametrize("surface", ["rusanov", "hll"])
def test_euler2d_linearised_flux_decouples_on_y_uniform_fields(surface):
    rho0, v1, v2, p0 = 1.2, 0.35, -0.2, 0.9
    n_base = 4
    c = np.sqrt(GAMMA * p0 / rho0)
    u0 = np.array([rho0, rho0 * v1, rho0 * v2, p0 / (GAMMA - 1) + 0.5 * rho0 * (v1 * v1 + v2 * v2)])
    lam, R, Ri = _char_basis(_fd_jacobian(_euler_flux_x_2d, u0), c, v1)
    d = _dissipation(surface, lam, v1, c)
    Cm, Dm = _advection_parts(n_base)
    m = _mesh(2, "euler", surface, n_base)
    n, nv, npe = m.shape
    lv = m.leaves()
    # 2D node q = 4 j + i (x fastest); max_level 0, so the finest-grid origin is the base cell
    ix = np.asarray(lv["fx"])
    iy = np.asarray(lv["fy"])
    U0 = np.broadcast_to(u0[None, :, None], m.shape).copy()
    J = np.zeros((n_base, nv, 4, n_base, nv, 4))
    for cx in range(n_base):
        for v in range(nv):
            for i in range(4):
                d_ = np.zeros(m.shape)
                d_[ix == cx, v, i::4] = 1.0          # constant in y: every row j, every cell of column cx
                out = _ddir(m, U0, d_)
                # the image must be y-uniform as well
                o4 = out.reshape(n, nv, 4, 4)        # [cell][var][j][i]
                assert np.abs(o4 - o4[:, :, :1, :]).max() < 1e-8 * max(1.0, np.abs(o4).max())
                for cx2 in range(n_base):
                    sel = (ix == cx2) & (iy == 0)
                    J[cx2, :, :, cx, v, i] = o4[sel][0, :, 0, :]
    Jc = np.einsum("kv,evifuj,ul->ekiflj", Ri, J, R)
    scale = np.abs(Jc).max()
    for k in range(nv):
        for l in range(nv):
            blk = Jc[:, k, :, :, l, :].reshape(n_base * 4, n_base * 4)
            expect = lam[k] * Cm + d[k] * Dm if k == l else np.zeros_like(blk)
            assert np.abs(blk - expect).max() < 1e-8 * scale, (k, l, np.abs(blk - expect).max())
