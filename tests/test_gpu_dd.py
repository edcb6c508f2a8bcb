"""GPU parity of the spatial domain decomposition (include/perk.h perk_dd_*):
sub-domains of a P-way E-weighted split held in one process on one GPU (perk_dd_group_step, the
in-process form) against the undecomposed CUDA path and against the oracle.

* the device split equals the host perk_dd_split of the same leaves (bit-exact owners);
* every sub-domain's lists are the undecomposed lists restricted to its owned elements / faces with
  an owned side (bit-exact), the owned ranges tile the mesh, send list of p to q == receive list of q
  from p;
* states: the gathered owned rows equal the undecomposed run BITWISE (every owned cell sees the same
  arithmetic on the same inputs) and the oracle within 1e-10 -- Euler (P-ERK2 and P-ERK3), Navier-Stokes
  (BR1: viscous-flux traces exchanged), re-meshes (complete state gathered first), P = 2, 3, 4, 8;
* one rank per process (DistributedPerk, torch.distributed): 2 processes on this GPU with the gloo
  backend (buffers staged through host memory; no kernel waits on another process).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from oracle import tableau as T
from gpu_util import TOL, gpu_state_numpy, rel_err_per_var

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _single(w, family=None):
    from paper_2403_05144_b200 import Perk
    return Perk(w.problem, w.level_map, w.S, w.E, family=family, max_cells=w.problem["max_cells"])


def _group(w, P, family=None):
    from paper_2403_05144_b200 import DomainGroup
    return DomainGroup(w.problem, w.level_map, w.S, w.E, P, family=family, max_cells=w.problem["max_cells"])


def _check_lists(g, single):
    """owned / face restrictions of the undecomposed lists, tiling ranges, matching send / recv lists"""
    from paper_2403_05144_b200.perk import dd_split
    leaves = single.leaves()
    wts = np.array(single.E, np.int64)[leaves["member"]]
    ranges = g.ranges()
    P = g.nranks
    owner_host = dd_split(wts, P)
    first = 0
    for p, (f, c) in enumerate(ranges):
        assert f == first and np.all(owner_host[f:f + c] == p)
        first += c
    assert first == single.n_cells
    owner = owner_host
    faces = {k: single.faces(k)[0] for k in ("interfaces", "mortars")}
    for p, part in enumerate(g.parts):
        lst, seg = part.list("elements")
        lo, sego = single.list("elements")
        assert np.array_equal(lst, lo[owner[lo] == p])
        li, segi = part.list("interfaces")
        lio, _ = single.list("interfaces")
        rec = faces["interfaces"]
        keep = (owner[rec[lio, 0]] == p) | (owner[rec[lio, 1]] == p)
        assert np.array_equal(li, lio[keep])
        lm, _ = part.list("mortars")
        lmo, _ = single.list("mortars")
        recm = faces["mortars"]
        keep = (owner[recm[lmo, 0]] == p) | (owner[recm[lmo, 1]] == p) | (owner[recm[lmo, 2]] == p)
        assert np.array_equal(lm, lmo[keep])
        for q in range(P):
            if q == p:
                continue
            snd = part.dd_list(q, 0)
            rcv = g.parts[q].dd_list(p, 1)
            assert np.array_equal(snd, rcv)
            assert np.all(owner[snd] == p)


def _run_compare(w, P, steps, family=None, remesh=None):
    fam = family or T.family(w.S, w.E, w.alpha_rule)
    ora = O.OracleMesh(w.problem, w.level_map, fam)
    single = _single(w, family)
    g = _group(w, P, family)
    _check_lists(g, single)
    Uo = ora.initial_state(w.ic)
    Us = single.initial_state(w.ic)
    Ug = g.initial_state(w.ic)
    done, k = 0, 0
    while done < steps:
        n = min(remesh or steps, steps - done)
        ora.step(Uo, w.dt, n)
        single.step(Us, w.dt, n)
        g.step(Ug, w.dt, n)
        done += n
        if remesh and done < steps:
            k += 1
            lm = w.level_map_seq(k)
            new = O.OracleMesh(w.problem, lm, fam)
            Uo = O.transfer(ora, new, Uo)
            ora = new
            single.repartition(lm, Us)
            g.repartition(lm, Ug)
            g.sync()
            _check_lists(g, single)
    torch.cuda.synchronize()
    g.sync()
    single.sync()
    S = gpu_state_numpy(single, Us)
    G = g.gather(Ug)
    assert np.array_equal(G, S), np.abs(G - S).max()          # bitwise the undecomposed path
    assert rel_err_per_var(G, Uo).max() <= TOL
    ev_g, _ = g.counters()
    ev_s, _ = single.counters()
    assert ev_g == ev_s                                        # the sub-domains' evaluations add up
    g.close()
    single.close()


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_dd_euler_cfg3_structure(P):
    w = W.make(3, n_base=16)
    _run_compare(w, P, 20)


def test_dd_euler_full_cfg3_mesh():
    w = W.make(3)
    _run_compare(w, 4, 3)


def test_dd_perk3():
    from workloads import perk3 as P3
    w = W.make(3, n_base=16)
    _run_compare(w, 3, 15, family=P3.family3(w.S, w.E))


@pytest.mark.parametrize("P", [2, 4])
def test_dd_navier_stokes(P):
    w = W.make(5, n_base=32)
    _run_compare(w, P, 6)


def test_dd_remesh_cfg4():
    w = W.make(4, n_base=16, max_level=3, widths=(0.3, 0.15, 0.06))
    w.S, w.E = 16, [4, 6, 10, 16]
    w.problem = dict(w.problem, max_cells=4 * W.configs.count_leaves(w))
    _run_compare(w, 3, 20, remesh=5)


def test_dd_device_owner_matches_host_split():
    from paper_2403_05144_b200.perk import dd_split
    w = W.make(5)
    single = _single(w)
    wts = np.array(w.E, np.int64)[single.leaves()["member"]]
    for P in (2, 3, 8):
        g = _group(w, P)
        owner = dd_split(wts, P)
        for p, (f, c) in enumerate(g.ranges()):
            assert c == int((owner == p).sum()) and (c == 0 or owner[f] == p)
        g.close()


def test_dd_rejects():
    from paper_2403_05144_b200 import Perk, PerkError
    w = W.make(3, n_base=8)
    for bad in (dict(rank=2, nranks=2), dict(rank=0, nranks=9)):
        with pytest.raises(PerkError) as ei:
            Perk(w.problem, w.level_map, w.S, w.E, **bad)
        assert ei.value.code == -1
    w1 = W.make(1)
    with pytest.raises(PerkError) as ei:
        Perk(w1.problem, w1.level_map, w1.S, w1.E, rank=0, nranks=2)
    assert ei.value.code == -6
    p = Perk(w.problem, w.level_map, w.S, w.E, rank=0, nranks=2)
    U = p.initial_state(w.ic)
    with pytest.raises(PerkError) as ei:
        p.step(U, w.dt)
    assert ei.value.code == -6
    with pytest.raises(PerkError) as ei:
        p.set_shock_capturing(W.configs.SHOCK_CAPTURING)
    assert ei.value.code == -6


@pytest.mark.parametrize("cfg", ["3", "5"])
def test_dd_two_processes_gloo(cfg):
    """one sub-domain per process (DistributedPerk) on this GPU, gloo transport through host memory"""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr=127.0.0.1", f"--master-port={port}",
                          os.path.join(ROOT, "tools", "dd_multiproc.py"), cfg],
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert res["bitwise_equal_single"], res
    assert res["max_rel_err_oracle"] <= TOL, res
    assert res["evals_sum_equal"], res
