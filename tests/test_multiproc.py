"""The N > 1 path of bench.py on CPU: world_size-2 gloo process group (127.0.0.1), replicas with the
per-rank step time reduced by MAX and the whole-job value = all ranks' units / the slowest time
("replicas only", no data-path collective)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    ws_, rank_, local_ = bench._dist()
    assert (ws_, rank_, local_) == (ws, rank, rank)
    ms_local = [0.70, 0.95][rank]                          # rank 1 is the slow replica
    ms = bench._max_over_ranks(torch, dist, ws, torch.device("cpu"), ms_local)
    val = bench.replica_value(ws, 713596.0, ms)
    out[rank] = (ms, val)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_max_timing():
    ws = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, _free_port(), out), nprocs=ws, join=True)
    for r in range(ws):
        ms, val = out[r]
        assert ms == 0.95                                  # both ranks see the max
        assert abs(val - 2 * 713596.0 / 0.95e-3) < 1e-6 * val


def test_single_rank_is_identity():
    import bench
    assert bench._max_over_ranks(torch, None, 1, None, 1.25) == 1.25
    assert bench.replica_value(1, 1000.0, 2.0) == 500000.0
