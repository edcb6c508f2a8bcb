"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol that
include/perk.h declares, and its host-only tableau builder agrees with the oracle's exact one."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import tableau as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2403_05144_b200 import build
    build.build()
    from paper_2403_05144_b200 import perk
    return perk


def _header_functions():
    src = open(os.path.join(ROOT, "include", "perk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*\*?\s*(\w+)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(lib):
    L = lib.lib()
    names = _header_functions()
    assert len(names) >= 20
    for nm in names:
        assert hasattr(L, nm), nm
    assert sorted(lib.exported_symbols()) == names


def test_no_oracle_dependency():
    """the product package never imports / links the oracle (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_2403_05144_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "perk_oracle" not in txt, f


@pytest.mark.parametrize("S,E", [(8, [4, 8]), (16, [4, 8, 16]), (28, [4, 6, 10, 16, 28]), (32, [4, 8, 16, 32])])
def test_library_tableau_matches_oracle(lib, S, E):
    t = lib.tableau_p2(S, E)
    fam = T.family(S, E, "taylor")
    for i in range(S):
        assert t.c[i] == fam["c_f"][i]
        for r in range(len(E)):
            want = fam["asub_f"][r][i]
            assert abs(t.a_sub[r][i] - want) <= 1e-14 * abs(want)   # double recursion vs exact rationals


def test_library_tableau_disk_rows(lib):
    """disk polynomial coefficients passed explicitly reproduce the printed table (P:l.535-561)."""
    fam = T.family(16, [8, 16], "disk")
    rows = [[float(a[k]) for k in range(17)] if len(a) == 17 else [float(a[k]) for k in range(len(a))]
            for a in fam["alpha"]]
    t = lib.tableau_p2(16, [8, 16], rows)
    for i in range(16):
        for r in range(2):
            want = fam["asub_f"][r][i]
            assert abs(t.a_sub[r][i] - want) <= 1e-14 * abs(want)


def test_invalid_tableau_rejected(lib):
    with pytest.raises(lib.PerkError):
        lib.tableau_p2(8, [8, 4])
    with pytest.raises(lib.PerkError):
        lib.tableau_p2(8, [4, 9])


def test_product_path_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import workloads as W
    w = W.make(1)
    with pytest.raises(RuntimeError):
        lib.Perk(w.problem, w.level_map, w.S, w.E)


@pytest.mark.parametrize("pattern", ["alternating", "early", [[1, 3, 6, 8], [1, 2, 4, 5, 8], "standard"]])
@pytest.mark.parametrize("c_S", [0.5, 1.0, 2.0 / 3.0])
def test_library_pattern_tableau_matches_oracle(lib, pattern, c_S):
    """stage patterns and Heun / Ralston weights: the library's masks, c, b and chain
    coefficients agree with the oracle's exact ones (independent implementations)"""
    from fractions import Fraction as Fr
    S, E = 8, [4, 5, 8]
    cS = Fr(2, 3) if abs(c_S - 2 / 3) < 1e-12 else Fr(c_S)
    fam = T.family(S, E, "taylor", pattern=pattern, c_S=cS)
    t = lib.tableau_p2(S, E, pattern=pattern, c_S=c_S)
    masks = fam["active_mask"] or [0] * 3
    assert [t.active[r] for r in range(3)] == masks
    for i in range(S):
        assert abs(t.c[i] - fam["c_f"][i]) <= 1e-16 and abs(t.b[i] - fam["b_f"][i]) <= 1e-16
        for r in range(3):
            want = fam["asub_f"][r][i]
            assert (want == 0) == (t.a_sub[r][i] == 0) and abs(t.a_sub[r][i] - want) <= 1e-14 * abs(want)


def test_invalid_patterns_rejected(lib):
    for pat in ([[1, 2, 8], [1, 3, 4, 5, 8], "standard"],      # member 0 holds 3 stages, E = 4
                [[2, 3, 4, 8], [1, 2, 4, 5, 8], "standard"],   # stage 1 missing
                [[1, 2, 3, 4], [1, 2, 4, 5, 8], "standard"]):  # stage S missing
        with pytest.raises(lib.PerkError):
            lib.tableau_p2(8, [4, 5, 8], pattern=pat)


def test_pattern_mask_behind_the_abi(lib):
    """perk_pattern_mask (the stage-pattern rule lives in the library, not the binding) against the
    oracle's stage sets, every S <= 40 and 2 <= E <= S, plus the printed S = 6, E = 4 sets
    (P:l.655-700: alternating {1,3,4,6}, early-shared {1,2,3,6})"""
    assert lib.pattern_mask(6, 4, "alternating") == 0b101101
    assert lib.pattern_mask(6, 4, "early") == 0b100111
    for S in range(2, 41):
        for E in range(2, S + 1):
            for pat in ("standard", "early", "alternating"):
                want = sum(1 << (i - 1) for i in T.pattern_stages(S, E, pat))
                assert lib.pattern_mask(S, E, pat) == want, (S, E, pat)
    assert lib.pattern_mask(8, 4, [1, 3, 6, 8]) == 0b10100101
    for bad in ([1, 3, 3, 8], [2, 3, 6, 8], [1, 3, 6, 7], [1, 3, 8], [1, 3, 6, 9]):
        with pytest.raises(lib.PerkError):
            lib.pattern_mask(8, 4, bad)
    with pytest.raises(lib.PerkError):
        lib.pattern_mask(8, 9, "standard")
