"""Multi-process host logic of the scenario sharder on CPU (gloo, world size 2):
contiguous scenario blocks, one int64 SUM all-reduce of the tally vector, max-over-ranks
timing.  The per-rank compute here is the oracle (no GPU in this container); the GPU path
uses the same module with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import dilu_inputs as di
import oracle
from paper_2503_05130_b200 import dist as ddist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    ddist.init("gloo")
    wl = di.c4(n_scenarios=12, T=120)
    lo, hi = ddist.block(wl.S, rank, world)
    _, tot = oracle.run(wl.shard(rank, world))
    assert wl.shard(rank, world).S == hi - lo
    t = torch.from_numpy(tot.copy())
    ddist.allreduce_tallies(t)
    mx = ddist.allreduce_max(float(rank + 1))
    ddist.barrier()
    out[rank] = (t.numpy().tolist(), mx)
    dist.destroy_process_group()


def test_block_partition():
    for n in (1, 7, 4096):
        for w in (1, 2, 3, 8):
            blocks = [ddist.block(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_world2_allreduce_matches_single_process():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    _, ref = oracle.run(di.c4(n_scenarios=12, T=120))
    for r in range(2):
        tally, mx = out[r]
        assert np.array_equal(np.array(tally, dtype=np.int64), ref)
        assert mx == 2.0
