"""Thin ctypes binding of libperk_b200.so (include/perk.h) -- argument marshalling only.

Every step of the P-ERK hot path (mesh/list rebuild, fluxes, volume integral, stage
combination, re-mesh transfer) runs in the CUDA kernels behind the C ABI.  PyTorch is used for
device memory and the current CUDA stream.  There is no CPU fallback: if the shared library is
missing or CUDA is unavailable, constructing a `Perk` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PERK_LIB_PATH") or os.path.join(HERE, "lib", "libperk_b200.so")   # env: A/B builds

EQ = {"advection": 0, "euler": 1, "navier_stokes": 2}
VOL = {"weak": 0, "fluxdiff": 1}
SURF = {"upwind": 0, "rusanov": 1, "hll": 2}
KIND = {"elements": 0, "interfaces": 1, "mortars": 2, "boundaries": 3}
ERRORS = {-1: "EINVAL", -2: "EUNBALANCED", -3: "ECAPACITY", -4: "ECUDA", -5: "ENOTINIT", -6: "EUNSUPPORTED"}
NP = 4
NKINDS = 7   # PERK_NUM_KERNEL_KINDS: surface, volume+stage, mesh, transfer, BR1 traces, BR1 gradients,
             # shock-capturing blending factors


class PerkError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class perk_problem(C.Structure):
    _fields_ = [("dim", C.c_int32), ("equation", C.c_int32), ("volume", C.c_int32), ("surface", C.c_int32),
                ("n_base", C.c_int32 * 2), ("max_level", C.c_int32), ("periodic", C.c_int32 * 2), ("_pad", C.c_int32),
                ("domain_lo", C.c_double * 2), ("domain_hi", C.c_double * 2), ("gamma", C.c_double),
                ("prandtl", C.c_double), ("mu", C.c_double), ("adv_velocity", C.c_double),
                ("bc_state", C.c_double * 4), ("max_cells", C.c_int64)]


class perk_tableau(C.Structure):
    _fields_ = [("S", C.c_int32), ("R", C.c_int32), ("E", C.c_int32 * 8), ("c", C.c_double * 64),
                ("b", C.c_double * 64), ("a_sub", (C.c_double * 64) * 8), ("active", C.c_uint64 * 8)]


class perk_amr(C.Structure):
    _fields_ = [("indicator", C.c_int32), ("variable", C.c_int32), ("base_level", C.c_int32),
                ("med_level", C.c_int32), ("max_level", C.c_int32), ("_pad", C.c_int32),
                ("med_threshold", C.c_double), ("max_threshold", C.c_double), ("alpha_max", C.c_double),
                ("alpha_min", C.c_double), ("f_wave", C.c_double)]


INDICATOR = {"hennemann_gassner": 0, "lohner": 1, "enstrophy": 2}
AMR_VARIABLE = {"rho": 0, "p": 1, "rho_p": 2, "v_x": 3, "v_y": 4}


def amr_params(a: dict) -> perk_amr:
    """perk_amr from a dict: indicator, variable, base/med/max_level, med/max_threshold,
    alpha_max (default 0.5), alpha_min (0.001), f_wave (0.2)"""
    s = perk_amr()
    s.indicator = INDICATOR[a["indicator"]]
    s.variable = AMR_VARIABLE[a.get("variable", "rho")]
    s.base_level, s.med_level, s.max_level = a["base_level"], a["med_level"], a["max_level"]
    s.med_threshold, s.max_threshold = a["med_threshold"], a["max_threshold"]
    s.alpha_max, s.alpha_min = a.get("alpha_max", 0.5), a.get("alpha_min", 0.001)
    s.f_wave = a.get("f_wave", 0.2)
    return s


class perk_shock_capturing(C.Structure):
    _fields_ = [("variable", C.c_int32), ("smooth", C.c_int32), ("alpha_max", C.c_double),
                ("alpha_min", C.c_double), ("alpha_fixed", C.c_double)]


def sc_params(sc: dict) -> perk_shock_capturing:
    """problem["shock_capturing"]: variable (AMR variable name, default rho_p), alpha_max (0.5), alpha_min
    (0.001), smooth (True), alpha_fixed (None = the Hennemann-Gassner indicator)"""
    s = perk_shock_capturing()
    s.variable = AMR_VARIABLE[sc.get("variable", "rho_p")]
    s.smooth = int(bool(sc.get("smooth", True)))
    s.alpha_max, s.alpha_min = sc.get("alpha_max", 0.5), sc.get("alpha_min", 0.001)
    af = sc.get("alpha_fixed")
    s.alpha_fixed = -1.0 if af is None else float(af)
    return s


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
        L.perk_alpha_taylor.argtypes = [i32, C.POINTER(dbl)]
        L.perk_tableau_p2.argtypes = [i32, i32, C.POINTER(i32), C.POINTER(dbl), C.POINTER(perk_tableau)]
        L.perk_tableau_p2_ex.argtypes = [i32, i32, C.POINTER(i32), C.POINTER(dbl), C.POINTER(C.c_uint64), dbl,
                                         C.POINTER(perk_tableau)]
        L.perk_pattern_mask.argtypes = [i32, i32, i32, C.POINTER(i32), i32, C.POINTER(C.c_uint64)]
        L.perk_init.argtypes = [C.POINTER(P), C.POINTER(perk_problem), P, C.POINTER(perk_tableau), P]
        L.perk_init_dd.argtypes = [C.POINTER(P), C.POINTER(perk_problem), P, C.POINTER(perk_tableau), P, i32, i32]
        L.perk_dd_split.argtypes = [i64, P, i32, P]
        L.perk_dd_info.argtypes = [P, C.POINTER(i32), C.POINTER(i32), C.POINTER(i64), C.POINTER(i64)]
        L.perk_dd_counts.argtypes = [P, i32, i32, P, P]
        L.perk_dd_get_list.argtypes = [P, i32, i32, P, i64, C.POINTER(i64)]
        L.perk_dd_stage.argtypes = [P, P, dbl, i32, i32]
        L.perk_dd_pack.argtypes = [P, P, i32, i32, i32, P]
        L.perk_dd_unpack.argtypes = [P, P, i32, i32, i32, P]
        L.perk_dd_exchange.argtypes = [P, P, P, P, i32, i32]
        L.perk_dd_group_step.argtypes = [P, i32, P, dbl]
        L.perk_debug_jitter.argtypes = [C.c_uint32]
        L.perk_destroy.argtypes = [P]
        L.perk_set_stream.argtypes = [P, P]
        L.perk_step.argtypes = [P, P, dbl]
        L.perk_run_host.argtypes = [P, P, dbl, i64]
        L.perk_repartition.argtypes = [P, P, P]
        L.rhs_eval.argtypes = [P, P, C.c_uint32, P]
        L.perk_num_cells.argtypes = [P, C.POINTER(i64)]
        L.perk_num_faces.argtypes = [P, C.POINTER(i64)]
        L.perk_node_coords.argtypes = [P, P]
        L.perk_get_leaves.argtypes = [P, P, P, P, P, i64]
        L.perk_get_faces.argtypes = [P, i32, P, P, i64, C.POINTER(i64)]
        L.perk_get_list.argtypes = [P, i32, P, i64, P]
        L.perk_get_count_active.argtypes = [P, i32, P]
        L.perk_get_halo_counts.argtypes = [P, P]
        L.perk_get_face_table.argtypes = [P, P, i64]
        L.perk_get_counters.argtypes = [P, C.POINTER(i64), C.POINTER(i64)]
        L.perk_sync.argtypes = [P]
        L.perk_last_error.argtypes = [P]
        L.perk_last_error.restype = C.c_char_p
        L.perk_profile_step.argtypes = [P, P, dbl, P, P]
        L.perk_time_kernels.argtypes = [P, P, dbl, C.c_uint32, i32, C.POINTER(C.c_float)]
        L.perk_time_kernels_ex.argtypes = [P, P, dbl, C.c_uint32, i32, P, i64, C.POINTER(C.c_float)]
        L.perk_profile_repartition.argtypes = [P, P, P, P, P]
        L.perk_launches_per_step.argtypes = [P, C.POINTER(i32)]
        L.perk_amr_indicator.argtypes = [P, P, C.POINTER(perk_amr), P]
        L.perk_amr_adapt.argtypes = [P, P, C.POINTER(perk_amr), P]
        L.perk_amr_launches.argtypes = [P, C.POINTER(i32)]
        L.perk_set_shock_capturing.argtypes = [P, C.POINTER(perk_shock_capturing)]
        L.perk_sc_alpha.argtypes = [P, P, P, P]
        _lib = L
    return _lib


def build_flags() -> dict:
    """the library's build configuration (perk_build_flags): BR1 variants"""
    f = int(lib().perk_build_flags())
    return {"br1_dv": bool(f & 1), "br1_fused": bool(f & 2)}


def exported_symbols():
    return ["perk_alpha_taylor", "perk_tableau_p2", "perk_tableau_p2_ex", "perk_init", "perk_destroy", "perk_set_stream", "perk_step",
            "perk_run_host", "perk_repartition", "rhs_eval", "perk_num_cells", "perk_num_faces", "perk_node_coords",
            "perk_get_leaves", "perk_get_faces", "perk_get_list", "perk_get_count_active", "perk_get_counters",
            "perk_sync", "perk_last_error", "perk_profile_step", "perk_time_kernels", "perk_profile_repartition",
            "perk_launches_per_step", "perk_amr_indicator", "perk_amr_adapt", "perk_amr_launches",
            "perk_set_shock_capturing", "perk_sc_alpha", "perk_pattern_mask", "perk_get_halo_counts", "perk_time_kernels_ex",
            "perk_init_dd", "perk_dd_split", "perk_dd_info", "perk_dd_counts", "perk_dd_get_list", "perk_dd_stage",
            "perk_dd_pack", "perk_dd_unpack", "perk_dd_exchange", "perk_dd_group_step", "perk_debug_jitter",
            "perk_build_flags", "perk_get_face_table"]


PATTERNS = {"standard": 0, "early": 1, "alternating": 2}


def pattern_mask(S: int, E: int, pattern) -> int:
    """Evaluated-stage bitmask (bit i-1 = stage i) of a member with E evaluations, computed by the
    library (perk_pattern_mask, include/perk.h): "standard", "early", "alternating" or an explicit
    iterable of stages."""
    m = C.c_uint64()
    if isinstance(pattern, str):
        if pattern not in PATTERNS:
            raise PerkError(-1, f"unknown stage pattern {pattern!r}")
        _check(None, lib().perk_pattern_mask(int(S), int(E), PATTERNS[pattern], None, 0, C.byref(m)))
    else:
        st = [int(i) for i in pattern]
        arr = (C.c_int32 * max(len(st), 1))(*st)
        _check(None, lib().perk_pattern_mask(int(S), int(E), 3, arr, len(st), C.byref(m)))
    return int(m.value)


def tableau_p2(S: int, E, alpha_rows=None, pattern=None, c_S: float = 0.5) -> perk_tableau:
    """P-ERK2 family via the library (C recursion).  alpha_rows: R rows of S+1 coefficients; default
    the Taylor rule alpha_k = 1/k! (BASELINE.json cfg 1), also built by the library.  pattern: None /
    "standard", a pattern name for every member, or one name / stage list per member;
    c_S: 1/2 standard, 1 Heun, 2/3 Ralston (P:l.439-442)."""
    E = [int(e) for e in E]
    R = len(E)
    al = np.zeros((R, S + 1))
    for r, e in enumerate(E):
        ek = max(0, min(e, S))          # out-of-range E is rejected by the library below
        if alpha_rows is None:
            row = (C.c_double * (ek + 1))()
            _check(None, lib().perk_alpha_taylor(ek, row))
            al[r, : ek + 1] = np.frombuffer(row, dtype=np.float64)
        else:
            n = min(len(alpha_rows[r]), S + 1)
            al[r, :n] = alpha_rows[r][:n]
    al = np.ascontiguousarray(al)
    t = perk_tableau()
    Ea = (C.c_int32 * R)(*E)
    act = None
    if pattern is not None and pattern != "standard":
        pats = pattern if isinstance(pattern, (list, tuple)) and len(pattern) == R and \
            not all(isinstance(x, int) for x in pattern) else [pattern] * R
        masks = [pattern_mask(S, e, pt) for e, pt in zip(E, pats)]
        if masks != [pattern_mask(S, e, "standard") for e in E]:
            act = (C.c_uint64 * R)(*masks)
    _check(None, lib().perk_tableau_p2_ex(S, R, Ea, al.ctypes.data_as(C.POINTER(C.c_double)), act, float(c_S),
                                          C.byref(t)))
    return t


def tableau_from(family: dict) -> perk_tableau:
    """Marshal an explicit family (e.g. a P-ERK3 family of workloads/perk3.py: c_f, b_f, asub_f, E) into
    the C struct; the library validates it at perk_init."""
    t = perk_tableau()
    S, E = int(family["S"]), [int(e) for e in family["E"]]
    t.S, t.R = S, len(E)
    for i in range(S):
        t.c[i] = family["c_f"][i]
        t.b[i] = family["b_f"][i]
    for r, e in enumerate(E):
        t.E[r] = e
        for i in range(S):
            t.a_sub[r][i] = family["asub_f"][r][i]
    for r, m in enumerate(family.get("active_mask") or []):
        t.active[r] = int(m)
    return t


def _check(h, rc):
    if rc != 0:
        msg = lib().perk_last_error(h).decode() if h else ""
        raise PerkError(rc, msg)


def _problem_struct(p: dict, max_cells: int) -> perk_problem:
    s = perk_problem()
    s.dim = p["dim"]
    s.equation = EQ[p["equation"]]
    s.volume = VOL[p["volume"]]
    s.surface = SURF[p["surface"]]
    s.n_base[0], s.n_base[1] = p["n_base"]
    s.max_level = p["max_level"]
    s.periodic[0], s.periodic[1] = [int(x) for x in p["periodic"]]
    s.domain_lo[0], s.domain_lo[1] = p["domain_lo"]
    s.domain_hi[0], s.domain_hi[1] = p["domain_hi"]
    s.gamma, s.prandtl, s.mu, s.adv_velocity = p["gamma"], p["prandtl"], p["mu"], p["adv_velocity"]
    for k, v in enumerate(p["bc_state"]):
        s.bc_state[k] = v
    s.max_cells = int(max_cells)
    return s


def _ptr(t):
    return C.c_void_p(t.data_ptr())


class Perk:
    """One P-ERK multirate DGSEM context on the current CUDA device (all work on the current stream)."""

    def __init__(self, problem: dict, level_map, S: int, E, alpha_rows=None, max_cells=None, stream=None,
                 family=None, pattern=None, c_S: float = 0.5, rank: int = 0, nranks: int = 1):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("CUDA device required: libperk_b200 has no CPU path")
        self.torch = torch
        self.problem = problem
        self.dim = problem["dim"]
        self.nv = problem["nv"]
        self.npe = NP ** self.dim
        self.S = S
        self.E = list(E)
        self.R = len(self.E)
        self.max_cells = int(max_cells or problem["max_cells"])
        self._tab = tableau_p2(S, self.E, alpha_rows, pattern, c_S) if family is None else tableau_from(family)
        self._prob = _problem_struct(problem, self.max_cells)
        lm = self._to_dev_u8(level_map)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        h = C.c_void_p()
        self.rank, self.nranks = int(rank), int(nranks)
        rc = lib().perk_init_dd(C.byref(h), C.byref(self._prob), _ptr(lm), C.byref(self._tab),
                                C.c_void_p(self.stream.cuda_stream), self.rank, self.nranks)
        self.h = h
        if rc != 0:
            msg = lib().perk_last_error(h).decode() if h else ""
            if h:
                lib().perk_destroy(h)
                self.h = None
            raise PerkError(rc, msg)
        if problem.get("shock_capturing") is not None:
            self.set_shock_capturing(problem["shock_capturing"])

    def set_shock_capturing(self, sc):
        """sc: dict (see sc_params) or None (off)"""
        self._sc = None if sc is None else sc_params(sc)
        _check(self.h, lib().perk_set_shock_capturing(self.h, None if sc is None else C.byref(self._sc)))

    def sc_alpha(self, U):
        """shock-capturing blending factors of U: (raw, smoothed) device tensors of n_cells doubles"""
        raw = self.torch.zeros(self.max_cells, dtype=self.torch.float64, device="cuda")
        sm = self.torch.zeros(self.max_cells, dtype=self.torch.float64, device="cuda")
        _check(self.h, lib().perk_sc_alpha(self.h, _ptr(U), _ptr(raw), _ptr(sm)))
        n = self.n_cells
        return raw[:n], sm[:n]

    def _to_dev_u8(self, level_map):
        torch = self.torch
        if isinstance(level_map, torch.Tensor):
            return level_map.to(device="cuda", dtype=torch.uint8).contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(level_map, dtype=np.uint8))).cuda()

    def close(self):
        if getattr(self, "h", None):
            lib().perk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state ----
    @property
    def n_cells(self) -> int:
        n = C.c_int64()
        _check(self.h, lib().perk_num_cells(self.h, C.byref(n)))
        return n.value

    def face_counts(self) -> dict:
        a = (C.c_int64 * 3)()
        _check(self.h, lib().perk_num_faces(self.h, a))
        return {"interfaces": a[0], "mortars": a[1], "boundaries": a[2]}

    def alloc_state(self):
        return self.torch.zeros((self.max_cells, self.nv, self.npe), dtype=self.torch.float64, device="cuda")

    def node_coords(self):
        torch = self.torch
        xy = torch.zeros((self.max_cells, self.dim, self.npe), dtype=torch.float64, device="cuda")
        _check(self.h, lib().perk_node_coords(self.h, _ptr(xy)))
        n = self.n_cells
        return xy[:n, 0] if self.dim == 1 else xy[:n]

    def initial_state(self, ic):
        """U (capacity rows) with the first n_cells rows = ic evaluated at this mesh's nodes."""
        xy = self.node_coords().cpu().numpy()
        U0 = ic(xy) if self.dim == 1 else ic(xy[:, 0, :], xy[:, 1, :])
        U0 = np.ascontiguousarray(np.moveaxis(np.asarray(U0, np.float64), 0, 1))
        U = self.alloc_state()
        U[: U0.shape[0]] = self.torch.from_numpy(U0).cuda()
        return U

    # ---- the hot path ----
    def step(self, U, dt: float, nsteps: int = 1):
        assert U.is_cuda and U.dtype == self.torch.float64 and U.is_contiguous()
        for _ in range(nsteps):
            _check(self.h, lib().perk_step(self.h, _ptr(U), float(dt)))

    def run_host(self, U_host, dt: float, nsteps: int = 1):
        """End-to-end call with a host (ideally pinned) float64 tensor of n_cells rows."""
        assert not U_host.is_cuda and U_host.dtype == self.torch.float64 and U_host.is_contiguous()
        _check(self.h, lib().perk_run_host(self.h, C.c_void_p(U_host.data_ptr()), float(dt), int(nsteps)))

    def repartition(self, level_map, U):
        lm = self._to_dev_u8(level_map)
        _check(self.h, lib().perk_repartition(self.h, _ptr(lm), _ptr(U)))
        self._keep = lm   # keep the map alive until the stream has consumed it

    def amr_indicator(self, U, amr: dict):
        """per-leaf AMR indicator (device tensor of n_cells doubles)"""
        ind = self.torch.zeros(self.max_cells, dtype=self.torch.float64, device="cuda")
        a = amr_params(amr)
        _check(self.h, lib().perk_amr_indicator(self.h, _ptr(U), C.byref(a), _ptr(ind)))
        return ind[: self.n_cells]

    def amr_adapt(self, U, amr: dict, out=None):
        """next finest-grid level map (device uint8 tensor (nfy, nfx)); asynchronous"""
        p = self.problem
        L = p["max_level"]
        shape = (p["n_base"][1] << L, p["n_base"][0] << L)
        if out is None:
            out = self.torch.zeros(shape, dtype=self.torch.uint8, device="cuda")
        a = amr_params(amr)
        _check(self.h, lib().perk_amr_adapt(self.h, _ptr(U), C.byref(a), _ptr(out)))
        return out

    def amr_launches(self) -> int:
        n = C.c_int32()
        _check(self.h, lib().perk_amr_launches(self.h, C.byref(n)))
        return n.value

    def rhs(self, U, mask=None):
        mask = (1 << self.R) - 1 if mask is None else int(mask)
        dU = self.torch.zeros_like(U)
        _check(self.h, lib().rhs_eval(self.h, _ptr(U), mask, _ptr(dU)))
        return dU

    def sync(self):
        _check(self.h, lib().perk_sync(self.h))

    # ---- introspection ----
    def leaves(self) -> dict:
        n = self.n_cells
        fx = np.zeros(n, np.int32)
        fy = np.zeros(n, np.int32)
        lev = np.zeros(n, np.uint8)
        mem = np.zeros(n, np.int32)
        _check(self.h, lib().perk_get_leaves(self.h, fx.ctypes.data, fy.ctypes.data, lev.ctypes.data, mem.ctypes.data, n))
        return dict(fx=fx, fy=fy, level=lev, member=mem)

    def faces(self, kind: str):
        k = KIND[kind]
        width = {1: 3, 2: 5, 3: 2}[k]
        n = self.face_counts()[kind]
        rec = np.zeros(max(n, 1) * width, np.int32)
        mem = np.zeros(max(n, 1), np.int32)
        ln = C.c_int64()
        _check(self.h, lib().perk_get_faces(self.h, k, rec.ctypes.data, mem.ctypes.data, max(n, 1), C.byref(ln)))
        return rec[: n * width].reshape(n, width), mem[:n]

    def list(self, kind: str):
        k = KIND[kind]
        n = self.n_cells if k == 0 else self.face_counts()[kind]
        lst = np.zeros(max(n, 1), np.int32)
        seg = np.zeros(self.R + 1, np.int64)
        _check(self.h, lib().perk_get_list(self.h, k, lst.ctypes.data, max(n, 1), seg.ctypes.data))
        return lst[: int(seg[-1])], seg      # a sub-domain's lists hold only its owned items

    def count_active(self, kind: str):
        out = np.zeros(self.S, np.int32)
        _check(self.h, lib().perk_get_count_active(self.h, KIND[kind], out.ctypes.data))
        return out

    def face_table(self):
        """per element face neighbours of the fused BR1 pass: int32 [n_cells][4][2] (include/perk.h)"""
        out = np.zeros(8 * max(self.n_cells, 1), np.int32)
        _check(self.h, lib().perk_get_face_table(self.h, out.ctypes.data, out.size))
        return out[: 8 * self.n_cells].reshape(self.n_cells, 4, 2)

    def halo_counts(self):
        """BR1 / shock-capturing halo items per stage: dict kind -> array of S counts"""
        out = np.zeros(3 * self.S, np.int32)
        _check(self.h, lib().perk_get_halo_counts(self.h, out.ctypes.data))
        return {"elements": out[: self.S], "interfaces": out[self.S: 2 * self.S], "mortars": out[2 * self.S:]}

    def counters(self):
        ev, st = C.c_int64(), C.c_int64()
        _check(self.h, lib().perk_get_counters(self.h, C.byref(ev), C.byref(st)))
        return ev.value, st.value

    def launches_per_step(self) -> int:
        n = C.c_int32()
        _check(self.h, lib().perk_launches_per_step(self.h, C.byref(n)))
        return n.value

    def profile_step(self, U, dt):
        ms = (C.c_float * NKINDS)()
        nl = (C.c_int32 * NKINDS)()
        _check(self.h, lib().perk_profile_step(self.h, _ptr(U), float(dt), ms, nl))
        return list(ms), list(nl)

    def time_kernels(self, U, dt, kinds, reps=10, flush=None):
        """device ms per step of only the kernels of `kinds` (0 surface, 1 volume+stage, 4/5 BR1),
        launched as perk_step does (graph + programmatic launches); timing only, U is garbage after.
        flush: a device tensor overwritten between the replays (L2 flush), or None"""
        mask = 0
        for k in kinds:
            mask |= 1 << k
        ms = C.c_float()
        if flush is None:
            _check(self.h, lib().perk_time_kernels(self.h, _ptr(U), float(dt), mask, int(reps), C.byref(ms)))
        else:
            nbytes = flush.numel() * flush.element_size()
            _check(self.h, lib().perk_time_kernels_ex(self.h, _ptr(U), float(dt), mask, int(reps), _ptr(flush),
                                                      int(nbytes), C.byref(ms)))
        return ms.value

    def profile_repartition(self, level_map, U):
        lm = self._to_dev_u8(level_map)
        ms = (C.c_float * NKINDS)()
        nl = (C.c_int32 * NKINDS)()
        _check(self.h, lib().perk_profile_repartition(self.h, _ptr(lm), _ptr(U), ms, nl))
        return list(ms), list(nl)

    @property
    def tableau(self) -> dict:
        t = self._tab
        return dict(S=t.S, R=t.R, E=list(t.E[: t.R]), c=list(t.c[: t.S]),
                    a_sub=[list(t.a_sub[r][: t.S]) for r in range(t.R)])


# ------------------------------------------------------------------------------------------------
# spatial domain decomposition (include/perk.h perk_dd_*) -- marshalling only
# ------------------------------------------------------------------------------------------------
def dd_split(weights, nranks: int):
    """the library's E-weighted contiguous split (host function perk_dd_split): owner rank per leaf"""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.int32))
    out = np.zeros(max(len(w), 1), np.int32)
    _check(None, lib().perk_dd_split(len(w), w.ctypes.data, int(nranks), out.ctypes.data))
    return out[: len(w)]


def _dd_info(p):
    r, n, f, c = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
    _check(p.h, lib().perk_dd_info(p.h, C.byref(r), C.byref(n), C.byref(f), C.byref(c)))
    return r.value, n.value, f.value, c.value


def _dd_counts(p, peer, what):
    snd = np.zeros(p.S, np.int32)
    rcv = np.zeros(p.S, np.int32)
    _check(p.h, lib().perk_dd_counts(p.h, int(peer), int(what), snd.ctypes.data, rcv.ctypes.data))
    return snd, rcv


def _dd_list(p, peer, direction):
    n = C.c_int64()
    buf = np.zeros(max(p.max_cells, 1), np.int32)
    _check(p.h, lib().perk_dd_get_list(p.h, int(peer), int(direction), buf.ctypes.data, len(buf), C.byref(n)))
    return buf[: n.value]


Perk.dd_info = lambda self: _dd_info(self)
Perk.dd_counts = lambda self, peer, what: _dd_counts(self, peer, what)
Perk.dd_list = lambda self, peer, direction: _dd_list(self, peer, direction)


class DomainGroup:
    """All sub-domains of an nranks-way split held by this process on the current device and stream
    (perk_init_dd + perk_dd_group_step): the in-process form of the multi-GPU decomposition, used to
    prove it on one GPU.  Every sub-domain keeps a full-size state whose owned rows are its own."""

    def __init__(self, problem: dict, level_map, S: int, E, nranks: int, **kw):
        self.parts = [Perk(problem, level_map, S, E, rank=p, nranks=nranks, **kw) for p in range(nranks)]
        self.nranks = nranks
        self.torch = self.parts[0].torch

    def initial_state(self, ic):
        return [p.initial_state(ic) for p in self.parts]

    def step(self, Us, dt, nsteps: int = 1):
        arr = (C.c_void_p * self.nranks)(*[u.data_ptr() for u in Us])
        hs = (C.c_void_p * self.nranks)(*[p.h.value for p in self.parts])
        for _ in range(nsteps):
            _check(self.parts[0].h, lib().perk_dd_group_step(hs, self.nranks, arr, float(dt)))

    def ranges(self):
        return [_dd_info(p)[2:] for p in self.parts]

    def gather(self, Us):
        """the global state: each sub-domain's owned rows (numpy)"""
        n = self.parts[0].n_cells
        out = np.zeros((n,) + tuple(Us[0].shape[1:]))
        for p, U in zip(self.parts, Us):
            f, c = _dd_info(p)[2:]
            out[f:f + c] = U[f:f + c].cpu().numpy()
        return out

    def allgather(self, Us):
        """make every sub-domain's state complete (before perk_repartition / perk_amr_*)"""
        for p, U in zip(self.parts, Us):
            f, c = _dd_info(p)[2:]
            for V in Us:
                if V is not U:
                    V[f:f + c].copy_(U[f:f + c])

    def repartition(self, level_map, Us):
        self.allgather(Us)
        for p, U in zip(self.parts, Us):
            p.repartition(level_map, U)

    def counters(self):
        ev = st = 0
        for p in self.parts:
            e, s_ = p.counters()
            ev += e
            st = max(st, s_)
        return ev, st

    def sync(self):
        for p in self.parts:
            p.sync()

    def close(self):
        for p in self.parts:
            p.close()


class DistributedPerk:
    """One sub-domain per process (rank = torch.distributed rank): per stage the library's stage
    launches and pack / unpack kernels, with the blocks moved by torch.distributed point-to-point
    (NCCL on GPUs; with the gloo backend the buffers are staged through host memory, which is how
    the path is exercised with several processes on one GPU)."""

    def __init__(self, problem: dict, level_map, S: int, E, dist, **kw):
        self.dist = dist
        self.rank, self.nranks = dist.get_rank(), dist.get_world_size()
        self.p = Perk(problem, level_map, S, E, rank=self.rank, nranks=self.nranks, **kw)
        self.torch = self.p.torch
        self.ns = problem["equation"] == "navier_stokes"
        self.host_staged = dist.get_backend() != "nccl"
        self._setup()
        dist.barrier()   # every rank's communicator is up before the first point-to-point batch

    def _setup(self):
        """per peer and exchange kind: per-stage block counts (synchronising; once per mesh)"""
        p = self.p
        self.row = {0: p.nv * p.npe, 1: 48}
        self.cnt = {}
        self.peers = []
        for q in range(self.nranks):
            if q == self.rank:
                continue
            c0 = _dd_counts(p, q, 0)
            if c0[0].max() > 0 or c0[1].max() > 0:
                self.peers.append(q)
            self.cnt[(q, 0)] = c0
            if self.ns:
                self.cnt[(q, 1)] = _dd_counts(p, q, 1)
        nmax = max([int(max(c[0].max(), c[1].max())) for c in self.cnt.values()] + [1])
        T = self.torch
        self.sbuf = {q: T.empty(nmax * 64, dtype=T.float64, device="cuda") for q in self.peers}
        self.rbuf = {q: T.empty(nmax * 64, dtype=T.float64, device="cuda") for q in self.peers}

    def initial_state(self, ic):
        return self.p.initial_state(ic)

    def _exchange(self, U, i, what):
        T, dist, p = self.torch, self.dist, self.p
        lib_ = lib()
        for q in self.peers:
            _check(p.h, lib_.perk_dd_pack(p.h, _ptr(U), i, what, q, _ptr(self.sbuf[q])))
        ops, host = [], {}
        for q in self.peers:
            ns_, nr_ = int(self.cnt[(q, what)][0][i - 1]), int(self.cnt[(q, what)][1][i - 1])
            sb = self.sbuf[q][: ns_ * self.row[what]]
            rb = self.rbuf[q][: nr_ * self.row[what]]
            if self.host_staged:
                sb, rb_h = sb.cpu(), T.empty(rb.numel(), dtype=T.float64)
                host[q] = rb_h
                rb = rb_h
            if ns_:
                ops.append(dist.P2POp(dist.isend, sb, q))
            if nr_:
                ops.append(dist.P2POp(dist.irecv, rb, q))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for q in self.peers:
            nr_ = int(self.cnt[(q, what)][1][i - 1])
            if not nr_:
                continue
            if self.host_staged:
                self.rbuf[q][: nr_ * self.row[what]].copy_(host[q])
            _check(p.h, lib_.perk_dd_unpack(p.h, _ptr(U), i, what, q, _ptr(self.rbuf[q])))

    def step(self, U, dt, nsteps: int = 1):
        p = self.p
        lib_ = lib()
        for _ in range(nsteps):
            for i in range(1, p.S + 1):
                if self.ns:
                    _check(p.h, lib_.perk_dd_stage(p.h, _ptr(U), float(dt), i, 0))
                    self._exchange(U, i, 1)
                _check(p.h, lib_.perk_dd_stage(p.h, _ptr(U), float(dt), i, 1))
                self._exchange(U, i, 0)

    def owned(self):
        return _dd_info(self.p)[2:]

    def allgather(self, U):
        """complete state on every rank (before perk_repartition / perk_amr_*): owned row ranges"""
        T, dist = self.torch, self.dist
        f, c = self.owned()
        meta = T.tensor([f, c], dtype=T.int64, device="cuda" if not self.host_staged else "cpu")
        allm = [T.zeros_like(meta) for _ in range(self.nranks)]
        dist.all_gather(allm, meta)
        for q, m in enumerate(allm):
            fq, cq = int(m[0]), int(m[1])
            blk = U[fq:fq + cq].contiguous()
            if self.host_staged:
                blk = blk.cpu()
            dist.broadcast(blk, src=q)
            if q != self.rank:
                U[fq:fq + cq].copy_(blk)

    def repartition(self, level_map, U):
        self.allgather(U)
        self.p.repartition(level_map, U)
        self._setup()

    def counters(self):
        return self.p.counters()

    def close(self):
        self.p.close()
