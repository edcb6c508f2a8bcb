"""Helpers for the GPU parity tests: build the oracle and the CUDA path on the same seeded
workload (workloads/), compare lists bitwise and states per conserved variable."""
import numpy as np

from oracle import oracle as O
from oracle import tableau as T

TOL = 1e-10   # BASELINE.json north_star: <= 1e-10 max relative fp64 state error per conserved variable


def rel_err_per_var(Ug, Uo):
    """||U_gpu,v - U_ora,v||_inf / ||U_ora,v||_inf per variable v."""
    out = []
    for v in range(Uo.shape[1]):
        den = np.abs(Uo[:, v]).max()
        out.append(np.abs(Ug[:, v] - Uo[:, v]).max() / (den if den > 0 else 1.0))
    return np.array(out)


def build_pair(w, problem=None, level_map=None, max_cells=None):
    from paper_2403_05144_b200 import Perk
    problem = problem or w.problem
    level_map = w.level_map if level_map is None else level_map
    fam = T.family(w.S, w.E, w.alpha_rule)
    ora = O.OracleMesh(problem, level_map, fam)
    gpu = Perk(problem, level_map, w.S, w.E, max_cells=max_cells or problem["max_cells"])
    return ora, gpu


def compare_mesh(ora, gpu, kinds=("elements", "interfaces", "mortars", "boundaries")):
    lo, lg = ora.leaves(), gpu.leaves()
    for k in ("fx", "fy", "level", "member"):
        assert np.array_equal(lo[k], lg[k]), k
    for kind in kinds:
        if kind != "elements":
            ro, mo = ora.faces(kind)
            rg, mg = gpu.faces(kind)
            assert np.array_equal(ro, rg), kind
            assert np.array_equal(mo, mg), kind
        lo_, so = ora.list(kind)
        lg_, sg = gpu.list(kind)
        assert np.array_equal(lo_, lg_), kind
        assert np.array_equal(so, sg), kind
        assert np.array_equal(ora.count_active(kind), gpu.count_active(kind)), kind


def gpu_state_numpy(gpu, U):
    n = gpu.n_cells
    return U[:n].cpu().numpy()


def expected_face_table(ora):
    """the fused BR1 pass's per element face neighbours (include/perk.h perk_get_face_table), written
    out from the oracle's face records: conforming {nb, -1}, small side {large, -2 / -3 (lower / upper
    half)}, large side {small_lo, small_hi}, boundary {-1, -4}; every face slot exactly once"""
    n = ora.n
    t = np.zeros((n, 4, 2), np.int32)
    seen = np.zeros((n, 4), np.int32)

    def put(e, f, a, b):
        t[e, f] = (a, b)
        seen[e, f] += 1

    for lo, hi, o in ora.faces("interfaces")[0]:
        put(lo, 2 * o, hi, -1)
        put(hi, 2 * o + 1, lo, -1)
    for large, s0, s1, o, side in ora.faces("mortars")[0]:
        put(large, 2 * o + side, s0, s1)
        put(s0, 2 * o + 1 - side, large, -2)
        put(s1, 2 * o + 1 - side, large, -3)
    for e, f in ora.faces("boundaries")[0]:
        put(e, f, -1, -4)
    assert (seen == 1).all(), "oracle face records do not cover every face slot once"
    return t
