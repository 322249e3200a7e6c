"""GPU: row strips of one image (BASELINE c3/c4), the multi-GPU split of a
single large image, run as "virtual strips" on one B200 (several strips on the same
device: the halo copies become device-local copies, the per-strip plans and windows are
exactly those of the multi-GPU run).

* the plan's explicit output window (crop=2) against the oracle on random cases;
* 2 / 4 / 8 strips of c3 and c4, stitched, against the reference's own output digests
  (tests/golden/digests.json, dilate and erode);
* the one-process-per-GPU driver (RankStrip: IPC handles + peer copies of the halo rows)
  with two processes sharing GPU 0, against the one-image result.
"""

import hashlib
import json
import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import cnaive

pytestmark = pytest.mark.gpu


def _digest(v, valid):
    return hashlib.sha256(np.ascontiguousarray(v, dtype=np.int32).tobytes()
                          + np.ascontiguousarray(valid, dtype=np.uint8).tobytes()).hexdigest()


def test_output_window_matches_oracle():
    """crop=2: output rows/cols [lo, lo+shape) of the dilation/erosion, any placement
    (inside, overlapping and outside the image), vs the full-range oracle result."""
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    rng = np.random.default_rng(11)
    for trial in range(24):
        H, W = (int(x) for x in rng.integers(20, 150, 2))
        my, mx = (int(x) for x in rng.integers(1, 14, 2))
        se = rng.integers(0, 8, (my, mx))
        sd = rng.random((my, mx)) < 0.7
        sd.flat[0] = True
        lo = (int(-(my // 2) + rng.integers(-2, 3)), int(-(mx // 2) + rng.integers(-2, 3)))
        img = rng.integers(0, 40, (H, W)).astype(np.uint8)
        mode = "erode" if trial % 2 else "dilate"
        fill = 39 if mode == "erode" else 0
        full, fvalid = cnaive.naive(img, None, se, sd, lo, erode=mode == "erode", crop=False, fill=fill)
        # full-range output index 0 <-> image index off (dilation: lo; erosion: -(lo + m - 1))
        off = lo if mode == "dilate" else (-(lo[0] + my - 1), -(lo[1] + mx - 1))
        wy0 = int(rng.integers(-my, H)), int(rng.integers(-mx, W))
        wsh = int(rng.integers(1, H + my)), int(rng.integers(1, W + mx))
        plan = MorphPlan(shape=(H, W), se_values=se, se_defined=sd, se_lo=lo, mode=mode, img_dtype=torch.uint8,
                         img_min=0, img_max=39, fill=fill, device=torch.device("cuda", 0), window=(wy0, wsh))
        out, valid = plan.execute(torch.from_numpy(img).cuda().unsqueeze(0))
        exp = np.full(wsh, fill, np.int32)
        expv = np.zeros(wsh, bool)
        for y in range(wsh[0]):
            fy = wy0[0] + y - off[0]
            if not 0 <= fy < full.shape[0]:
                continue
            xs = np.arange(wsh[1]) + wy0[1] - off[1]
            ok = (xs >= 0) & (xs < full.shape[1])
            exp[y, ok] = full[fy, xs[ok]]
            expv[y, ok] = fvalid[fy, xs[ok]]
        assert np.array_equal(out[0].cpu().numpy(), exp), trial
        assert np.array_equal(valid[0].cpu().numpy().astype(bool), expv), trial
        plan.close()


@pytest.mark.parametrize("name", ["c3", "c4"])
@pytest.mark.parametrize("nstrips", [2, 4, 8])
def test_virtual_strips_vs_reference_digests(name, nstrips):
    import torch
    from paper_2305_03018_b200 import workloads as W
    from paper_2305_03018_b200.strips import dilate_strips, erode_strips
    dg = json.loads((GOLDEN / "digests.json").read_text())[f"{name}_img0"]
    w = W.CONFIGS[name]()
    img = torch.from_numpy(w.images[0])
    sd = None if w.se_defined.all() else w.se_defined
    out, valid = dilate_strips(img, w.se_values, w.se_lo, devices=[0] * nstrips, se_defined=sd,
                               img_min=0, img_max=w.tonal_max)
    assert _digest(out.cpu().numpy(), valid.cpu().numpy()) == dg["dilate"]
    out, valid = erode_strips(img, w.se_values, w.se_lo, devices=[0] * nstrips, se_defined=sd,
                              img_min=0, img_max=w.tonal_max, l=w.tonal_max)
    assert _digest(out.cpu().numpy(), valid.cpu().numpy()) == dg["erode"]


def test_strips_small_uneven_and_more_strips_than_rows():
    """Strip counts that do not divide H, strips thinner than the SE, empty strips."""
    import torch
    from paper_2305_03018_b200.strips import dilate_strips
    rng = np.random.default_rng(4)
    img = rng.integers(0, 60, (37, 90)).astype(np.uint8)
    se = rng.integers(0, 5, (11, 7))
    ref, refv = cnaive.naive(img, None, se, None, (-5, -3), erode=False, crop=True, fill=0)
    for n in (3, 5, 16, 40):
        out, valid = dilate_strips(torch.from_numpy(img), se, (-5, -3), devices=[0] * n, img_min=0, img_max=59)
        assert np.array_equal(out.cpu().numpy(), ref), n
        assert np.array_equal(valid.cpu().numpy().astype(bool), refv), n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_03018_b200.strips import RankStrip
        torch.cuda.set_device(0)
        rng = np.random.default_rng(99)
        img = rng.integers(0, 16, (300, 257)).astype(np.uint8)
        se = np.zeros((41, 41), np.int64)
        sd = rng.random((41, 41)) < 0.5
        sd[20, 20] = True
        rs = RankStrip(rank=rank, world=world, shape=img.shape, se_values=se, se_defined=sd, se_lo=(-20, -20),
                       img_min=0, img_max=15, device=torch.device("cuda", 0))
        me = rs.me
        rs.load_own(torch.from_numpy(img[me.out0:me.out1]).cuda())
        torch.cuda.synchronize()
        dist.barrier()                         # every rank's own rows are in place
        s = torch.cuda.current_stream()
        rs.exchange_halos(s)
        out, valid = rs.execute(s)
        torch.cuda.synchronize()
        ok_window = np.array_equal(rs.window.cpu().numpy(), img[me.in0:me.in1])
        parts = [None] * world
        dist.all_gather_object(parts, (me.out0, out[0].cpu().numpy(), valid[0].cpu().numpy(), ok_window))
        dist.barrier()
        rs.close()
        if rank == 0:
            parts.sort(key=lambda t: t[0])
            full = np.concatenate([p[1] for p in parts])
            fv = np.concatenate([p[2] for p in parts]).astype(bool)
            ref, refv = cnaive.naive(img, None, se, sd, (-20, -20), erode=False, crop=True, fill=0)
            q.put(bool(all(p[3] for p in parts) and np.array_equal(full, ref) and np.array_equal(fv, refv)))
    finally:
        dist.destroy_process_group()


def test_rank_strips_ipc_halos_two_processes():
    """RankStrip (one process per GPU: IPC handles + peer copies of halo rows), here two
    processes sharing GPU 0 (they only copy from each other's buffers, no kernel waits on
    another process), stitched bit-exact."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5)
