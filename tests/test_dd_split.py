"""Host logic of the spatial domain decomposition (include/perk.h perk_dd_split):
the E-weighted split of the Morton-ordered leaves into contiguous rank ranges, on CPU (the library
loads without a GPU; no kernel runs here), and its use by a world_size-2 gloo process group (each
rank computes the split of the same mesh independently; the ranges must agree and tile the mesh).

The split is the build's design, not the paper's (the paper partitions by level only and says the
per-level lists need no exchange beyond standard RK, P:l.1258-1263): per-step work of a leaf is E of
its member, so the ranges are balanced in sum E (an equal-cell split is unbalanced under multirate)."""
import os
import socket

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from oracle import tableau as T

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    from paper_2403_05144_b200 import build
    build.build()
    from paper_2403_05144_b200 import perk
    return perk


def _leaf_weights(cfg, **kw):
    w = W.make(cfg, **kw)
    m = O.OracleMesh(w.problem, w.level_map, T.family(w.S, w.E, w.alpha_rule))
    mem = m.leaves()["member"]
    return np.array(w.E, np.int64)[mem]


def _check_split(wts, owner, P):
    n = len(wts)
    assert len(owner) == n
    assert np.all(np.diff(owner) >= 0) and owner.min() >= 0 and owner.max() <= P - 1   # contiguous ranges
    Wt = wts.sum()
    loads = np.array([wts[owner == p].sum() for p in range(P)])
    assert loads.sum() == Wt
    # midpoint rule: every rank's load is within one leaf weight of W / P
    assert np.abs(loads - Wt / P).max() <= wts.max() + 1e-9, (loads, Wt / P)
    return loads


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("cfg,kw", [(3, {}), (5, {"n_base": 64}), (4, {"n_base": 32})])
def test_split_balances_stage_evaluations(lib, P, cfg, kw):
    wts = _leaf_weights(cfg, **kw)
    owner = lib.dd_split(wts, P)
    loads = _check_split(wts, owner, P)
    if P > 1:
        # the equal-cell split of the same leaves is less balanced under multirate (the point of E weights)
        eq = np.minimum((np.arange(len(wts)) * P) // len(wts), P - 1)
        loads_eq = np.array([wts[eq == p].sum() for p in range(P)])
        assert loads.max() <= loads_eq.max()


def test_split_definition_and_edges(lib):
    # brute force of the definition on small random weights
    rng = np.random.default_rng(3)
    for _ in range(50):
        n, P = int(rng.integers(1, 40)), int(rng.integers(1, 9))
        wts = rng.integers(0, 33, n)
        owner = lib.dd_split(wts, P)
        Wt = int(wts.sum())
        pre = np.concatenate([[0], np.cumsum(wts)[:-1]])
        want = np.zeros(n, np.int64) if Wt == 0 else np.minimum((P * (2 * pre + wts)) // (2 * Wt), P - 1)
        assert np.array_equal(owner, want)
    assert len(lib.dd_split([], 4)) == 0
    for bad in (([1, -1], 2), ([1, 2], 0), ([1, 2], 9)):
        with pytest.raises(lib.PerkError):
            lib.dd_split(*bad)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2403_05144_b200 import perk
    wts = _leaf_weights(3)
    owner = perk.dd_split(wts, ws)
    mine = np.nonzero(owner == rank)[0]
    rng_ = torch.tensor([int(mine.min()), len(mine), int(wts[mine].sum())], dtype=torch.int64)
    allr = [torch.zeros_like(rng_) for _ in range(ws)]
    dist.all_gather(allr, rng_)
    h = torch.tensor([int(np.dot(owner, np.arange(len(owner)) % 7919))], dtype=torch.int64)
    allh = [torch.zeros_like(h) for _ in range(ws)]
    dist.all_gather(allh, h)
    out[rank] = ([r.tolist() for r in allr], [int(x) for x in allh], int(wts.sum()), len(wts))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_split_agrees_and_tiles():
    ws = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, _free_port(), out), nprocs=ws, join=True)
    r0, r1 = out[0], out[1]
    assert r0 == r1                                  # both ranks computed the same split
    ranges, hashes, Wt, n = r0
    assert len(set(hashes)) == 1
    assert ranges[0][0] == 0 and ranges[0][0] + ranges[0][1] == ranges[1][0]
    assert ranges[1][0] + ranges[1][1] == n          # contiguous, tiling
    assert abs(ranges[0][2] - ranges[1][2]) <= 2 * 16   # balanced within the largest leaf weight (E = 16)
    assert ranges[0][2] + ranges[1][2] == Wt
