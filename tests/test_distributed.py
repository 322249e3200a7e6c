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


def _window_worker(rank, world, port, mode, q):
    """Each rank computes ITS strip exactly as the product's per-strip plan does
    (strips.strip_plan_kwargs: image = the strip's input rows, output window = its owned
    rows): here the window is cut out of the oracle's full-range result on the strip
    rows, at the plan's window offset.  Stitched, it must equal the one-image result."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from oracle import cnaive
        from paper_2305_03018_b200 import sharding, strips as S
        rng = np.random.default_rng(321)
        H, W = 61, 37
        img = rng.integers(0, 40, (H, W)).astype(np.int32)
        se = rng.integers(0, 5, (11, 4))
        sd = rng.random((11, 4)) > 0.3
        sd[5, 1] = True
        lo = (-7, -1)       # SE not centred: asymmetric halos
        my, mx = se.shape
        plan = sharding.strips(H, world, lo[0], my, mode)
        me = plan[rank]
        local = torch.from_numpy(img[me.out0:me.out1].copy())
        window = sharding.exchange_halos(local, plan, rank).numpy()
        kw = S.strip_plan_kwargs(me, W)
        assert kw["shape"] == window.shape
        (wy, wx), (wh, ww) = kw["window"]
        erode = mode == "erode"
        fill = 99 if erode else 0
        full, fvalid = cnaive.naive(window, None, se, sd, lo, erode=erode, crop=False, fill=fill, threads=1)
        off_y = -(lo[0] + my - 1) if erode else lo[0]
        off_x = -(lo[1] + mx - 1) if erode else lo[1]
        mine = np.full((wh, ww), fill, np.int32)
        for y in range(wh):
            fy = wy + y - off_y
            if 0 <= fy < full.shape[0]:
                xs = np.arange(ww) + wx - off_x
                ok = (xs >= 0) & (xs < full.shape[1])
                mine[y, ok] = full[fy, xs[ok]]
        gathered = [None] * world
        dist.all_gather_object(gathered, (me.out0, mine))
        if rank == 0:
            stitched = np.concatenate([g[1] for g in sorted(gathered, key=lambda t: t[0])])
            ref, _ = cnaive.naive(img, None, se, sd, lo, erode=erode, crop=True, fill=fill)
            q.put(bool(np.array_equal(stitched, ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["dilate", "erode"])
def test_row_strip_plan_windows_bit_exact(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_window_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def _bench_worker(rank, world, port, q):
    """bench.py's multi-rank orchestration on CPU (gloo): rank-safe build, image shards,
    max-over-ranks timing, parity and image-count reductions."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        import bench
        from paper_2305_03018_b200 import build as B
        from paper_2305_03018_b200.sharding import shard_range
        B.build_rank_safe(rank, world)
        i0, i1 = shard_range(bench.N_IMAGES, rank, world)
        cpu = torch.device("cpu")
        ms = bench.over_ranks(10.0 + rank, "max", world, cpu)
        ok = bench.over_ranks(0 if rank == world - 1 else 1, "min", world, cpu)
        n = bench.over_ranks(i1 - i0, "sum", world, cpu)
        q.put((rank, ms, ok, n))
    finally:
        dist.destroy_process_group()


def test_bench_orchestration_gloo():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    for rank, ms, ok, n in res:
        assert ms == 10.0 + world - 1 and ok == 0 and n == 64


def test_reference_arm_is_time_bounded():
    """bench.py --impl reference: a driver-sized run (--steps 20) must not take steps x 17 s of
    host time; steps past the budget are skipped and the line says how many ran."""
    import bench
    res = bench.cpu_reference(steps=5, warmup=0, config="c1", budget_s=0.0)
    assert len(res["steps_s"]) == 1 and res["value"] > 0
    res = bench.cpu_reference(steps=3, warmup=1, config="c1", budget_s=600.0)
    assert len(res["steps_s"]) == 3 and res["kind"] == "port"
