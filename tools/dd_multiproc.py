"""One sub-domain per process (paper_2403_05144_b200.DistributedPerk) under torchrun: every rank steps
its part of a BASELINE-structured mesh with the library's stage launches and pack / unpack kernels,
the blocks moved by torch.distributed point-to-point; rank 0 then compares the gathered state with the
undecomposed CUDA path (bitwise) and with the oracle (<= 1e-10).  Used by tests/test_gpu_dd.py with
the gloo backend and 2 processes on one GPU (buffers staged through host memory, so no kernel waits on
another process); with NCCL and one GPU per rank it is the multi-GPU path of bench.py --gpus N.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port P \
      tools/dd_multiproc.py 3|5 [steps] [backend]
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import workloads as W  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    backend = sys.argv[3] if len(sys.argv) > 3 else "gloo"
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist.init_process_group(backend)
    from paper_2403_05144_b200 import DistributedPerk, Perk
    w = W.make(cfg, n_base=16 if cfg == 3 else 32)
    dp = DistributedPerk(w.problem, w.level_map, w.S, w.E, dist)
    U = dp.initial_state(w.ic)
    dp.step(U, w.dt, steps)
    torch.cuda.synchronize()
    dp.allgather(U)
    torch.cuda.synchronize()
    n = dp.p.n_cells
    G = U[:n].cpu().numpy()
    ev, _ = dp.counters()
    evs = torch.tensor([ev], dtype=torch.int64)
    alle = [torch.zeros_like(evs) for _ in range(ws)]
    dist.all_gather(alle, evs)
    if rank == 0:
        from oracle import oracle as O
        from oracle import tableau as T
        from gpu_util import rel_err_per_var
        single = Perk(w.problem, w.level_map, w.S, w.E)
        Us = single.initial_state(w.ic)
        single.step(Us, w.dt, steps)
        torch.cuda.synchronize()
        S = Us[:n].cpu().numpy()
        ora = O.OracleMesh(w.problem, w.level_map, T.family(w.S, w.E, w.alpha_rule))
        Uo = ora.initial_state(w.ic)
        ora.step(Uo, w.dt, steps)
        ev_s, _ = single.counters()
        print(json.dumps({"cfg": cfg, "ranks": ws, "steps": steps, "backend": backend, "cells": n,
                          "peers_of_rank0": dp.peers, "bitwise_equal_single": bool(np.array_equal(G, S)),
                          "max_abs_diff_single": float(np.abs(G - S).max()),
                          "max_rel_err_oracle": float(rel_err_per_var(G, Uo).max()),
                          "evals_sum_equal": int(sum(int(x) for x in alle)) == int(ev_s)}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
