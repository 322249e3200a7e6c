"""Row strips of ONE large image across GPUs (BASELINE c3/c4).

Each device owns the output rows [out0, out1) of its strip and holds the input
rows [in0, in1) those rows depend on: its own rows plus the SE-radius halos
owned by its neighbours (``sharding.strips``: the dependency cone of
dilate_naive / erode_naive, morphology.py:65-113).  The halos move by NVLink
peer copies (``fm_copy_peer`` = cudaMemcpyPeerAsync; a same-device copy when
strips share a GPU), then every device runs its own plan whose output WINDOW
is exactly its owned rows (``crop=2`` of fm_plan_desc), so nothing is computed
twice and the stitched result is bit-identical to the one-GPU result: each
output pixel depends only on f over x - B.  No collective is involved.

Two drivers share the geometry:

* :class:`StripPlan` — single process, many devices (``devices=[0, 1, ...]``;
  repeating a device runs "virtual strips" on one GPU, which is how the strip
  path is tested on a one-GPU box);
* :class:`RankStrip` — one process per GPU (torchrun): each rank keeps its
  strip buffer, exports it once as a CUDA IPC handle, maps its neighbours'
  buffers, and per step copies the halo rows straight out of their memory.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .engine import MorphPlan
from .sharding import Strip, strips


def _stream_ptr(stream):
    return ctypes.c_void_p(stream.cuda_stream)


def _copy_rows(dst: torch.Tensor, src: torch.Tensor, stream) -> None:
    """Peer copy of a contiguous row block (cudaMemcpyPeerAsync over NVLink between GPUs)."""
    assert dst.is_contiguous() and src.is_contiguous() and dst.numel() == src.numel() and dst.dtype == src.dtype
    nbytes = dst.numel() * dst.element_size()
    _lib.check(_lib.load().fm_copy_peer(ctypes.c_void_p(dst.data_ptr()), dst.device.index,
                                        ctypes.c_void_p(src.data_ptr()), src.device.index, nbytes,
                                        _stream_ptr(stream)))


def strip_plan_kwargs(st: Strip, W: int) -> dict:
    """Plan geometry of one strip: image = its input rows, output window = its owned rows."""
    return dict(shape=(st.in1 - st.in0, W), window=((st.out0 - st.in0, 0), (st.out1 - st.out0, W)))


class StripPlan:
    """Single-process row-strip pipeline over `devices` (one strip per entry)."""

    def __init__(self, *, shape, se_values, se_lo, devices, se_defined=None, mode="dilate",
                 img_dtype=torch.uint8, img_min=0, img_max=255, fill=0, out_dtype=torch.int32,
                 scratch_bytes=0):
        H, W = (int(s) for s in shape)
        se_values = np.asarray(se_values)
        self.H, self.W = H, W
        self.devices = [torch.device("cuda", int(d) if not isinstance(d, torch.device) else d.index)
                        for d in devices]
        self.plan_strips = strips(H, len(self.devices), int(se_lo[0]), se_values.shape[0], mode)
        self.img_dtype = img_dtype
        self.out_dtype = out_dtype
        self.plans, self.windows, self.streams = [], [], []
        for st, dev in zip(self.plan_strips, self.devices):
            if st.out1 <= st.out0:
                self.plans.append(None)
                self.windows.append(None)
                self.streams.append(None)
                continue
            self.plans.append(MorphPlan(se_values=se_values, se_lo=se_lo, se_defined=se_defined, mode=mode,
                                        img_dtype=img_dtype, img_min=img_min, img_max=img_max, fill=fill,
                                        batch=1, device=dev, out_dtype=out_dtype, scratch_bytes=scratch_bytes,
                                        **strip_plan_kwargs(st, W)))
            self.windows.append(torch.empty((st.in1 - st.in0, W), dtype=img_dtype, device=dev))
            self.streams.append(torch.cuda.Stream(dev))

    def load(self, img: torch.Tensor) -> None:
        """Place each strip's OWN rows on its device (from a host or device image [H, W])."""
        if tuple(img.shape) != (self.H, self.W) or img.dtype != self.img_dtype:
            raise ValueError(f"image must be [{self.H}, {self.W}] of {self.img_dtype}")
        for st, win, dev in zip(self.plan_strips, self.windows, self.devices):
            if win is None:
                continue
            win[st.out0 - st.in0: st.out1 - st.in0].copy_(img[st.out0:st.out1], non_blocking=False)
        for dev in set(self.devices):   # every own row in place before any halo copy reads it
            torch.cuda.synchronize(dev)

    def exchange_halos(self) -> None:
        """Halo rows from the strips that own them: peer copies, one per (neighbour, side)."""
        for dst_i, (dst, win) in enumerate(zip(self.plan_strips, self.windows)):
            if win is None:
                continue
            s = self.streams[dst_i]
            # the owners' rows must be in place (loaded / written on their streams)
            for src_i, (src, swin) in enumerate(zip(self.plan_strips, self.windows)):
                if src_i == dst_i or swin is None:
                    continue
                lo, hi = max(src.out0, dst.in0), min(src.out1, dst.in1)
                if hi <= lo:
                    continue
                if self.streams[src_i] is not None:
                    s.wait_stream(self.streams[src_i])
                _copy_rows(win[lo - dst.in0: hi - dst.in0], swin[lo - src.in0: hi - src.in0], s)

    def execute(self):
        """Run every strip on its device; returns per-strip (out, valid) of the owned rows."""
        res = []
        for plan, win, s in zip(self.plans, self.windows, self.streams):
            if plan is None:
                res.append(None)
                continue
            with torch.cuda.device(win.device):
                res.append(plan.execute(win.unsqueeze(0), stream=s))
        return res

    def synchronize(self) -> None:
        for s in self.streams:
            if s is not None:
                s.synchronize()

    def read_stats(self) -> float:
        self.synchronize()
        return max((p.read_stats() for p in self.plans if p is not None), default=0.0)

    def gather(self, parts, device=None):
        """Stitch per-strip results into full [H, W] tensors on `device` (default: the first)."""
        device = device or self.devices[0]
        self.synchronize()
        out = torch.empty((self.H, self.W), dtype=self.out_dtype, device=device)
        valid = torch.empty((self.H, self.W), dtype=torch.uint8, device=device)
        for st, pr in zip(self.plan_strips, parts):
            if pr is None:
                continue
            out[st.out0:st.out1].copy_(pr[0][0])
            valid[st.out0:st.out1].copy_(pr[1][0])
        return out, valid

    def run(self, img: torch.Tensor):
        self.load(img)
        self.exchange_halos()
        return self.gather(self.execute())

    def close(self) -> None:
        for p in self.plans:
            if p is not None:
                p.close()


def _strip_op(mode, img, se, se_lo, devices, se_defined, img_min, img_max, l, out_dtype):
    se = np.asarray(se.cpu() if isinstance(se, torch.Tensor) else se, dtype=np.int64)
    if se.ndim != 2:
        raise ValueError("row strips split 2-D images")
    if se_lo is None:
        se_lo = tuple(-(s // 2) for s in se.shape)
    if not isinstance(img, torch.Tensor):
        img = torch.from_numpy(np.ascontiguousarray(img))
    if img.dtype not in (torch.uint8, torch.uint16, torch.int32):
        img = img.to(torch.int32)
    if img_min is None or img_max is None:
        mn, mx = int(img.min().item()), int(img.max().item())
        img_min = mn if img_min is None else img_min
        img_max = mx if img_max is None else img_max
    fill = 0
    if mode == "erode":
        fill = int(img_max if l is None else l)
        if fill < img_max:
            raise ValueError(f"l={fill} below max value {img_max}")
    sp = StripPlan(shape=img.shape, se_values=se, se_lo=se_lo, devices=devices, se_defined=se_defined, mode=mode,
                   img_dtype=img.dtype, img_min=int(img_min), img_max=int(img_max), fill=fill, out_dtype=out_dtype)
    try:
        out = sp.run(img)
        sp.read_stats()
        return out
    finally:
        sp.close()


def dilate_strips(img, se, se_lo=None, *, devices, se_defined=None, img_min=None, img_max=None,
                  out_dtype=torch.int32):
    """Exact dilation of one 2-D image split into row strips over `devices` (dilate_fft
    semantics with crop=True: 0 / invalid where no pair exists); returns (values, validity)
    stitched on devices[0]."""
    return _strip_op("dilate", img, se, se_lo, devices, se_defined, img_min, img_max, None, out_dtype)


def erode_strips(img, se, se_lo=None, *, devices, l=None, se_defined=None, img_min=None, img_max=None,
                 out_dtype=torch.int32):
    """Exact erosion by row strips (erode_fft semantics: ``l`` where no pair exists, default
    the image maximum)."""
    return _strip_op("erode", img, se, se_lo, devices, se_defined, img_min, img_max, l, out_dtype)


class RankStrip:
    """One process per GPU (torchrun): this rank's strip, its plan, and IPC-mapped views of
    the neighbours' strip buffers for the per-step halo copies.

    Setup (not timed) exchanges CUDA IPC handles through the process group once
    (``all_gather_object``); each step is then ``exchange_halos()`` (peer copies out of the
    neighbours' memory on this rank's stream) + ``execute()``.  No collective on the data
    path.  The ranks' inputs must be in place before a step's halo copies (static inputs in
    the bench; a pipeline adds one barrier or IPC event per step)."""

    def __init__(self, *, rank, world, shape, se_values, se_lo, mode="dilate", se_defined=None,
                 img_dtype=torch.uint8, img_min=0, img_max=255, fill=0, out_dtype=torch.int32,
                 device=None, group=None):
        import torch.distributed as dist
        H, W = (int(s) for s in shape)
        se_values = np.asarray(se_values)
        self.rank, self.world, self.H, self.W = rank, world, H, W
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.plan_strips = strips(H, world, int(se_lo[0]), se_values.shape[0], mode)
        me = self.me = self.plan_strips[rank]
        self.window = torch.empty((me.in1 - me.in0, W), dtype=img_dtype, device=self.device)
        self.plan = MorphPlan(se_values=se_values, se_lo=se_lo, se_defined=se_defined, mode=mode,
                              img_dtype=img_dtype, img_min=img_min, img_max=img_max, fill=fill, batch=1,
                              device=self.device, out_dtype=out_dtype, **strip_plan_kwargs(me, W))
        self.esize = self.window.element_size()
        L = _lib.load()
        handle = (ctypes.c_char * 64)()
        off = ctypes.c_int64(0)
        _lib.check(L.fm_ipc_get_handle(ctypes.c_void_p(self.window.data_ptr()), handle, ctypes.byref(off)))
        mine = (bytes(handle), int(off.value), self.device.index)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.peers = {}     # src rank -> (mapped base pointer, offset, device)
        self.halos = []     # (src rank, row0, row1)
        for src in self.plan_strips:
            if src.rank == rank:
                continue
            lo, hi = max(src.out0, me.in0), min(src.out1, me.in1)
            if hi <= lo:
                continue
            if src.rank not in self.peers:
                h, o, d = allh[src.rank]
                ptr = ctypes.c_void_p()
                _lib.check(L.fm_ipc_open_handle(ctypes.create_string_buffer(h, 64), self.device.index,
                                                ctypes.byref(ptr)))
                self.peers[src.rank] = (ptr.value, o, d)
            self.halos.append((src.rank, lo, hi))

    def load_own(self, rows: torch.Tensor) -> None:
        me = self.me
        self.window[me.out0 - me.in0: me.out1 - me.in0].copy_(rows)

    def exchange_halos(self, stream) -> None:
        L = _lib.load()
        me = self.me
        row_b = self.W * self.esize
        for src_rank, lo, hi in self.halos:
            base, off, dev = self.peers[src_rank]
            src = self.plan_strips[src_rank]
            src_ptr = base + off + (lo - src.in0) * row_b
            dst_ptr = self.window.data_ptr() + (lo - me.in0) * row_b
            _lib.check(L.fm_copy_peer(ctypes.c_void_p(dst_ptr), self.device.index, ctypes.c_void_p(src_ptr),
                                      -1, (hi - lo) * row_b, _stream_ptr(stream)))

    def execute(self, stream, out=None, valid=None):
        return self.plan.execute(self.window.unsqueeze(0), out=out, valid=valid, stream=stream)

    def close(self) -> None:
        L = _lib.load()
        for base, _, _ in self.peers.values():
            L.fm_ipc_close_handle(ctypes.c_void_p(base))
        self.peers = {}
        self.plan.close()
