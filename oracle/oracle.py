"""ORACLE -- TEST INFRASTRUCTURE ONLY.  ctypes front end of oracle/perk_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this module.  It never imports paper_2403_05144_b200 and the CUDA path
never imports it.  See perk_oracle.c for the citations of each computation.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "perk_oracle.c")
# ORACLE_OMP=1: an OpenMP build (bitwise identical results, perk_oracle.c) for long full-run parity
# checks only; the tests and the CPU baseline use the serial build
OMP = os.environ.get("ORACLE_OMP") == "1"
LIB = os.path.join(HERE, "liboracle_omp.so" if OMP else "liboracle.so")

EQ = {"advection": 0, "euler": 1, "navier_stokes": 2}
VOL = {"weak": 0, "fluxdiff": 1}
SURF = {"upwind": 0, "rusanov": 1, "hll": 2, "ec": 3}
NP = 4


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc: -O2 -ffp-contract=off, no fast-math."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"] + \
              (["-fopenmp"] if OMP else []) + ["-o", LIB, SRC, "-lm"]
        subprocess.check_call(cmd)
    return LIB


class OraProblem(C.Structure):
    _fields_ = [("dim", C.c_int32), ("equation", C.c_int32), ("volume", C.c_int32), ("surface", C.c_int32),
                ("nbx", C.c_int32), ("nby", C.c_int32), ("max_level", C.c_int32), ("periodic", C.c_int32 * 2),
                ("lo", C.c_double * 2), ("hi", C.c_double * 2),
                ("gamma", C.c_double), ("prandtl", C.c_double), ("mu", C.c_double), ("adv", C.c_double),
                ("bc_state", C.c_double * 4)]


class OraTableau(C.Structure):
    _fields_ = [("S", C.c_int32), ("R", C.c_int32), ("E", C.c_int32 * 8), ("c", C.c_double * 64),
                ("b", C.c_double * 64), ("a1", (C.c_double * 64) * 8), ("asub", (C.c_double * 64) * 8),
                ("active", C.c_uint64 * 8)]


class OraAmr(C.Structure):
    _fields_ = [("indicator", C.c_int32), ("variable", C.c_int32), ("base_level", C.c_int32),
                ("med_level", C.c_int32), ("max_level", C.c_int32), ("_pad", C.c_int32),
                ("med_threshold", C.c_double), ("max_threshold", C.c_double),
                ("alpha_max", C.c_double), ("alpha_min", C.c_double), ("f_wave", C.c_double)]


class OraSC(C.Structure):
    _fields_ = [("variable", C.c_int32), ("smooth", C.c_int32), ("alpha_max", C.c_double),
                ("alpha_min", C.c_double), ("alpha_fixed", C.c_double)]


INDICATORS = {"hennemann_gassner": 0, "lohner": 1, "enstrophy": 2}
AMR_VARIABLES = {"rho": 0, "p": 1, "rho_p": 2, "v_x": 3, "v_y": 4}


def amr_struct(a: dict) -> OraAmr:
    s = OraAmr()
    s.indicator = INDICATORS[a["indicator"]]
    s.variable = AMR_VARIABLES[a.get("variable", "rho")]
    s.base_level, s.med_level, s.max_level = a["base_level"], a["med_level"], a["max_level"]
    s.med_threshold, s.max_threshold = a["med_threshold"], a["max_threshold"]
    s.alpha_max, s.alpha_min = a.get("alpha_max", 0.5), a.get("alpha_min", 0.001)
    s.f_wave = a.get("f_wave", 0.2)
    return s


def sc_struct(sc: dict) -> OraSC:
    """problem["shock_capturing"]: variable (AMR_VARIABLES name), alpha_max, alpha_min, smooth,
    alpha_fixed (None / negative = the indicator)"""
    s = OraSC()
    s.variable = AMR_VARIABLES[sc.get("variable", "rho_p")]
    s.smooth = int(sc.get("smooth", True))
    s.alpha_max, s.alpha_min = sc.get("alpha_max", 0.5), sc.get("alpha_min", 0.001)
    af = sc.get("alpha_fixed")
    s.alpha_fixed = -1.0 if af is None else af
    return s


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        ip = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        lp = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        up = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        L.ora_create.restype = P
        L.ora_create.argtypes = [C.POINTER(OraProblem), up, C.POINTER(OraTableau), C.c_char_p, C.c_int]
        L.ora_destroy.argtypes = [P]
        L.ora_num_cells.argtypes = [P]
        L.ora_face_counts.argtypes = [P, lp]
        L.ora_get_leaves.argtypes = [P, ip, ip, up, ip]
        L.ora_get_faces.argtypes = [P, C.c_int, ip, ip]
        L.ora_get_list.argtypes = [P, C.c_int, ip, lp]
        L.ora_count_active.argtypes = [P, C.c_int, ip]
        L.ora_node_coords.argtypes = [P, dp]
        L.ora_rhs.restype = C.c_int
        L.ora_rhs.argtypes = [P, dp, C.c_uint32, dp, C.c_int]
        L.ora_step.restype = C.c_int64
        L.ora_step.argtypes = [P, dp, C.c_double, C.c_int]
        L.ora_steps.restype = C.c_int64
        L.ora_steps.argtypes = [P, dp, C.c_double, C.c_int, C.c_int]
        L.ora_transfer.restype = C.c_int
        L.ora_transfer.argtypes = [P, P, dp, dp]
        L.ora_fv_rhs.argtypes = [C.c_int, dp, dp, dp, C.c_int, C.c_double]
        L.ora_fv_step.argtypes = [C.c_int, dp, ip, C.POINTER(OraTableau), dp, C.c_double, C.c_int, C.c_double]
        L.ora_ln_mean.restype = C.c_double
        L.ora_ln_mean.argtypes = [C.c_double, C.c_double]
        L.ora_flux_ranocha.argtypes = [dp, dp, C.c_int, C.c_double, dp]
        L.ora_num_flux_pub.argtypes = [P, dp, dp, C.c_int, dp]
        L.ora_get_basis.argtypes = [dp]
        L.ora_amr_indicator.restype = C.c_int
        L.ora_amr_indicator.argtypes = [P, dp, C.POINTER(OraAmr), dp]
        L.ora_amr_adapt.restype = C.c_int
        L.ora_amr_adapt.argtypes = [P, dp, C.POINTER(OraAmr), up]
        L.ora_amr_adapt_ind.restype = C.c_int
        L.ora_amr_adapt_ind.argtypes = [P, dp, C.POINTER(OraAmr), up]
        L.ora_set_shock_capturing.restype = C.c_int
        L.ora_set_shock_capturing.argtypes = [P, C.POINTER(OraSC)]
        L.ora_sc_alpha.restype = C.c_int
        L.ora_sc_alpha.argtypes = [P, dp, dp, dp]
        _lib = L
    return _lib


def problem_struct(p: dict) -> OraProblem:
    s = OraProblem()
    s.dim = p["dim"]
    s.equation = EQ[p["equation"]]
    s.volume = VOL[p["volume"]]
    s.surface = SURF[p["surface"]]
    s.nbx, s.nby = p["n_base"]
    s.max_level = p["max_level"]
    s.periodic[0], s.periodic[1] = [int(x) for x in p["periodic"]]
    s.lo[0], s.lo[1] = p["domain_lo"]
    s.hi[0], s.hi[1] = p["domain_hi"]
    s.gamma, s.prandtl, s.mu, s.adv = p["gamma"], p["prandtl"], p["mu"], p["adv_velocity"]
    for k, v in enumerate(p["bc_state"]):
        s.bc_state[k] = v
    return s


def tableau_struct(fam: dict) -> OraTableau:
    t = OraTableau()
    t.S, t.R = fam["S"], fam["R"]
    for r, E in enumerate(fam["E"]):
        t.E[r] = E
        for i in range(fam["S"]):
            t.a1[r][i] = fam["a1_f"][r][i]
            t.asub[r][i] = fam["asub_f"][r][i]
    b = fam.get("b_f") or [0.0] * (fam["S"] - 1) + [1.0]      # P-ERK2: b = e_S
    for i in range(fam["S"]):
        t.c[i] = fam["c_f"][i]
        t.b[i] = b[i]
    for r, m in enumerate(fam.get("active_mask") or []):      # stage patterns (0 = standard)
        t.active[r] = int(m)
    return t


def basis() -> dict:
    out = np.zeros(2 * NP + 7 * NP * NP)
    lib().ora_get_basis(out)
    names = ["xi", "w", "D", "Dhat", "Dsplit", "Plo", "Pup", "Rlo", "Rup"]
    res, o = {}, 0
    for nm in names:
        n = NP if nm in ("xi", "w") else NP * NP
        res[nm] = out[o:o + n].reshape((NP,) if n == NP else (NP, NP)).copy()
        o += n
    return res


def ln_mean(a, b):
    return lib().ora_ln_mean(a, b)


def flux_ranocha(uL, uR, orient, gamma=1.4):
    f = np.zeros(4)
    lib().ora_flux_ranocha(np.ascontiguousarray(uL, np.float64), np.ascontiguousarray(uR, np.float64),
                           orient, gamma, f)
    return f


class OracleMesh:
    """Oracle mesh + tableau context for one (problem, level map, family)."""

    KINDS = {"elements": 0, "interfaces": 1, "mortars": 2, "boundaries": 3}

    def __init__(self, problem: dict, level_map, fam: dict):
        self.problem = problem
        self.fam = fam
        self._p = problem_struct(problem)
        self._t = tableau_struct(fam)
        lm = np.ascontiguousarray(np.asarray(level_map, dtype=np.uint8).ravel())
        err = C.create_string_buffer(512)
        self.h = lib().ora_create(C.byref(self._p), lm, C.byref(self._t), err, 512)
        if not self.h:
            raise ValueError(err.value.decode())
        self.n = lib().ora_num_cells(self.h)
        if problem.get("shock_capturing") is not None:      # section 9 of perk_oracle.c
            self._sc = sc_struct(problem["shock_capturing"])
            rc = lib().ora_set_shock_capturing(self.h, C.byref(self._sc))
            if rc:
                raise ValueError("shock_capturing: " + ("unsupported problem" if rc == -2 else "invalid parameters"))
        self.nv = problem["nv"]
        self.npe = NP ** problem["dim"]

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_destroy(self.h)
            self.h = None

    @property
    def shape(self):
        return (self.n, self.nv, self.npe)

    def face_counts(self):
        out = np.zeros(3, np.int64)
        lib().ora_face_counts(self.h, out)
        return {"interfaces": int(out[0]), "mortars": int(out[1]), "boundaries": int(out[2])}

    def leaves(self):
        fx = np.zeros(self.n, np.int32)
        fy = np.zeros(self.n, np.int32)
        lev = np.zeros(self.n, np.uint8)
        mem = np.zeros(self.n, np.int32)
        lib().ora_get_leaves(self.h, fx, fy, lev, mem)
        return dict(fx=fx, fy=fy, level=lev, member=mem)

    def faces(self, kind: str):
        k = self.KINDS[kind]
        n = self.face_counts()[kind]
        width = {1: 3, 2: 5, 3: 2}[k]
        out = np.zeros(max(n, 1) * width, np.int32)
        mem = np.zeros(max(n, 1), np.int32)
        lib().ora_get_faces(self.h, k, out, mem)
        return out[: n * width].reshape(n, width), mem[:n]

    def list(self, kind: str):
        k = self.KINDS[kind]
        n = self.n if k == 0 else self.face_counts()[kind]
        lst = np.zeros(max(n, 1), np.int32)
        seg = np.zeros(self.fam["R"] + 1, np.int64)
        lib().ora_get_list(self.h, k, lst, seg)
        return lst[:n], seg

    def count_active(self, kind: str):
        out = np.zeros(self.fam["S"], np.int32)
        lib().ora_count_active(self.h, self.KINDS[kind], out)
        return out

    def node_coords(self):
        d = self.problem["dim"]
        xy = np.zeros(self.n * d * self.npe)
        lib().ora_node_coords(self.h, xy)
        return xy.reshape(self.n, d, self.npe) if d == 2 else xy.reshape(self.n, self.npe)

    def initial_state(self, ic) -> np.ndarray:
        xy = self.node_coords()
        if self.problem["dim"] == 1:
            U = ic(xy)                                  # (nv, n, npe)
        else:
            U = ic(xy[:, 0, :], xy[:, 1, :])
        return np.ascontiguousarray(np.moveaxis(np.asarray(U, np.float64), 0, 1))  # (n, nv, npe)

    def rhs(self, U, mask=None, mode=0):
        """dU = sum_{r in mask} I^(r) F(U).  mode 0 (default) is the definition (full F, then mask);
        mode 1 loops over the member lists and requires an upward-closed mask."""
        mask = (1 << self.fam["R"]) - 1 if mask is None else mask
        U = np.ascontiguousarray(U, np.float64)
        dU = np.zeros_like(U)
        if lib().ora_rhs(self.h, U.ravel(), mask, dU.ravel(), mode) != 0:
            raise ValueError("restricted mode needs an upward-closed partition mask")
        return dU

    def step(self, U, dt, nsteps=1, mode=1):
        """In place; returns element-RHS evaluations.  mode 1 = restricted (default), 0 = reference."""
        assert U.flags["C_CONTIGUOUS"] and U.dtype == np.float64
        return lib().ora_steps(self.h, U.reshape(-1), dt, nsteps, mode)


    def sc_alpha(self, U):
        """shock-capturing blending factors of state U: (raw indicator, smoothed), per leaf"""
        raw, sm = np.zeros(self.n), np.zeros(self.n)
        if lib().ora_sc_alpha(self.h, np.ascontiguousarray(U, np.float64).ravel(), raw, sm):
            raise ValueError("shock capturing is off")
        return raw, sm

    def amr_indicator(self, U, amr: dict):
        """per-leaf AMR indicator (section 8 of perk_oracle.c), canonical leaf order"""
        ind = np.zeros(self.n)
        a = amr_struct(amr)
        rc = lib().ora_amr_indicator(self.h, np.ascontiguousarray(U, np.float64).ravel(), C.byref(a), ind)
        if rc:
            raise ValueError(f"amr_indicator: {'unsupported problem' if rc == -2 else 'invalid parameters'}")
        return ind

    def amr_adapt(self, U, amr: dict, indicator=None):
        """new finest-grid level map (uint8, x fastest) from the controller + 2:1 balance; with
        `indicator` (per leaf, canonical order) the controller runs on those values instead of the
        oracle's own indicator of U (U is then unused)"""
        p = self.problem
        nf = [p["n_base"][0] << p["max_level"], p["n_base"][1] << p["max_level"]]
        lmap = np.zeros(nf[0] * nf[1], np.uint8)
        a = amr_struct(amr)
        if indicator is None:
            rc = lib().ora_amr_adapt(self.h, np.ascontiguousarray(U, np.float64).ravel(), C.byref(a), lmap)
        else:
            ind = np.ascontiguousarray(indicator, np.float64)
            assert ind.shape == (self.n,)
            rc = lib().ora_amr_adapt_ind(self.h, ind, C.byref(a), lmap)
        if rc:
            raise ValueError(f"amr_adapt: {'unsupported problem' if rc == -2 else 'invalid parameters'}")
        return lmap.reshape(nf[1], nf[0])


def transfer(old: OracleMesh, new: OracleMesh, U_old):
    U_new = np.zeros(new.shape)
    rc = lib().ora_transfer(old.h, new.h, np.ascontiguousarray(U_old).ravel(), U_new.reshape(-1))
    if rc != 0:
        raise ValueError(f"transfer failed ({rc})")
    return U_new


def fv_rhs(dx, U, kind=0, a=1.0):
    dx = np.ascontiguousarray(dx, np.float64)
    U = np.ascontiguousarray(U, np.float64)
    dU = np.zeros_like(U)
    lib().ora_fv_rhs(len(U), dx, U, dU, kind, a)
    return dU


def fv_step(dx, member, fam, U, dt, kind=0, a=1.0):
    dx = np.ascontiguousarray(dx, np.float64)
    member = np.ascontiguousarray(member, np.int32)
    U = np.array(U, dtype=np.float64, copy=True)
    t = tableau_struct(fam)
    lib().ora_fv_step(len(U), dx, member, C.byref(t), U, dt, kind, a)
    return U
