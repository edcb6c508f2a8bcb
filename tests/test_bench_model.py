"""bench.py's algorithmic-bytes model on CPU, with the oracle mesh standing in for the
device lists (same member-segment convention): the per-member form of the volume-kernel bytes equals
the stage-prefix form of round 1 (count_active of the elements), and the surface bytes follow the
face counts (every interface / mortar evaluated at stage 1, traces lazily formed only at stages
2 <= i <= S - E + 2)."""
import numpy as np
import pytest

import bench
import workloads as W
from oracle import oracle as O
from oracle import tableau as T


def _prefix_volume_bytes(count_el, S):
    B = 512
    tot = 3 * B * count_el[0]
    for i in range(2, S + 1):
        n = count_el[i - 1]
        newly = n - (count_el[i - 2] if i > 2 else 0)
        tot += 4 * B * n if i == S else 4 * B * newly + 5 * B * (n - newly)
    return tot


@pytest.mark.parametrize("cfg,kw", [(3, {}), (3, {"n_base": 16}), (4, {"n_base": 16})])
def test_volume_bytes_per_member_equals_prefix_form(cfg, kw):
    w = W.make(cfg, **kw)
    m = O.OracleMesh(w.problem, w.level_map, T.family(w.S, w.E, w.alpha_rule))
    b = bench.kernel_bytes_per_step(m, w)
    assert b["volume_stage"] == _prefix_volume_bytes(list(m.count_active("elements")), w.S)
    nif = m.face_counts()["interfaces"]
    nmo = m.face_counts()["mortars"]
    # stage 1 alone: every face with non-lazy traces (U_n): interface 2 x 128 + 2 x 128, mortar 3 x 128 + 3 x 128
    assert b["surface"] >= nif * 512 + nmo * 768
    assert b["surface"] <= w.S * (nif * (2 * 256 + 256) + nmo * (3 * 256 + 384))
