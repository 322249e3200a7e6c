"""Multi-GPU partitioning of the hot path (one process per GPU).

Two schemes, both without any collective on the data path:

* by image (c5): a batch of independent images is split into contiguous
  per-rank ranges — no exchange at all;
* by row strips (c3/c4, one large image): rank r owns output rows [r0, r1);
  its input window is widened by the SE's vertical reach and the missing
  rows (halos) are exchanged point-to-point with the ranks that own them
  (``torch.distributed`` send/recv: NVLink peer copies under NCCL, gloo on
  CPU for the tests).  Each output pixel depends only on f over x - B, so the
  stitched result is bit-identical to the single-GPU one.

The halo geometry restates the dependency cone of dilate_naive / erode_naive
(morphology.py:65-113): dilation output row y reads input rows
y - hi_y .. y - lo_y; erosion reads y + lo_y .. y + hi_y.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous split of n units: [start, end) for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


@dataclass(frozen=True)
class Strip:
    rank: int
    out0: int      # owned output rows [out0, out1)
    out1: int
    in0: int       # input rows needed [in0, in1)
    in1: int


def input_window(r0: int, r1: int, H: int, se_lo_y: int, se_h: int, mode: str) -> tuple[int, int]:
    """Input rows [i0, i1) that output rows [r0, r1) depend on (plus the owned rows)."""
    hi_y = se_lo_y + se_h - 1
    if mode == "dilate":
        a, b = r0 - hi_y, r1 - 1 - se_lo_y
    elif mode == "erode":
        a, b = r0 + se_lo_y, r1 - 1 + hi_y
    else:
        raise ValueError(f"unknown mode {mode!r}")
    i0 = max(0, min(r0, a))
    i1 = min(H, max(r1, b + 1))
    return i0, i1


def strips(H: int, world: int, se_lo_y: int, se_h: int, mode: str) -> list[Strip]:
    out = []
    for r in range(world):
        r0, r1 = shard_range(H, r, world)
        i0, i1 = input_window(r0, r1, H, se_lo_y, se_h, mode) if r1 > r0 else (r0, r0)
        out.append(Strip(r, r0, r1, i0, i1))
    return out


def halo_transfers(plan: list[Strip]) -> list[tuple[int, int, int, int]]:
    """(src, dst, row0, row1): rows of src's owned strip that dst needs and does not own."""
    xfers = []
    for dst in plan:
        for src in plan:
            if src.rank == dst.rank:
                continue
            lo = max(src.out0, dst.in0)
            hi = min(src.out1, dst.in1)
            if hi > lo:
                xfers.append((src.rank, dst.rank, lo, hi))
    return xfers


def exchange_halos(local_rows: torch.Tensor, plan: list[Strip], rank: int,
                   group=None) -> torch.Tensor:
    """Assemble rank's input window [in0, in1) from its own rows plus peers' halos.

    local_rows: [out1-out0, ...] rows this rank owns (any dtype, on the rank's device).
    Returns a tensor [in1-in0, ...] on the same device.
    """
    me = plan[rank]
    window = torch.empty((me.in1 - me.in0, *local_rows.shape[1:]), dtype=local_rows.dtype,
                         device=local_rows.device)
    if me.out1 > me.out0:
        window[me.out0 - me.in0: me.out1 - me.in0] = local_rows
    ops = []
    recv_bufs = []
    for src, dst, r0, r1 in halo_transfers(plan):
        if src == rank:
            ops.append(dist.P2POp(dist.isend, local_rows[r0 - me.out0: r1 - me.out0].contiguous(), dst, group))
        elif dst == rank:
            buf = torch.empty((r1 - r0, *local_rows.shape[1:]), dtype=local_rows.dtype, device=local_rows.device)
            recv_bufs.append((buf, r0))
            ops.append(dist.P2POp(dist.irecv, buf, src, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for buf, r0 in recv_bufs:
        window[r0 - me.in0: r0 - me.in0 + buf.shape[0]] = buf
    return window
