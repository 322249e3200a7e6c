"""CPU multi-process (gloo, world_size 2 and 3): the N>1 paths.

* row strips: each rank owns a strip of rows, exchanges SE-radius halos with
  torch.distributed P2P (the NCCL/NVLink path on the GPU box), computes its
  strip and the stitched result equals the single-process oracle bit for bit;
* by image: ranks take disjoint contiguous image ranges covering the batch.
The per-strip compute here is the oracle (C restatement) — this test checks
the partition and exchange logic, not the kernels.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from oracle import cnaive
        from paper_2305_03018_b200 import sharding
        rng = np.random.default_rng(123)
        H, W = 57, 41
        img = rng.integers(0, 50, (H, W)).astype(np.int32)
        se = rng.integers(0, 6, (9, 5))
        sd = rng.random((9, 5)) > 0.3
        sd[0, 0] = True
        lo = (-6, -2)
        plan = sharding.strips(H, world, lo[0], se.shape[0], mode)
        me = plan[rank]
        local = torch.from_numpy(img[me.out0:me.out1].copy())
        window = sharding.exchange_halos(local, plan, rank)
        assert np.array_equal(window.numpy(), img[me.in0:me.in1])
        erode = mode == "erode"
        out, valid = cnaive.naive(window.numpy(), None, se, sd, lo, erode=erode, crop=True,
                                  fill=99 if erode else 0, threads=1)
        mine = out[me.out0 - me.in0: me.out1 - me.in0]
        gathered = [None] * world
        dist.all_gather_object(gathered, (me.out0, mine))
        if rank == 0:
            full = np.concatenate([g[1] for g in sorted(gathered, key=lambda t: t[0])])
            ref, _ = cnaive.naive(img, None, se, sd, lo, erode=erode, crop=True, fill=99 if erode else 0)
            q.put(bool(np.array_equal(full, ref)))
        # by-image sharding
        from paper_2305_03018_b200.sharding import shard_range
        parts = [None] * world
        dist.all_gather_object(parts, shard_range(64, rank, world))
        if rank == 0:
            covered = sorted(i for s, e in parts for i in range(s, e))
            q.put(covered == list(range(64)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["dilate", "erode"])
def test_row_strip_halo_exchange_bit_exact(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
    assert q.get(timeout=10) is True
