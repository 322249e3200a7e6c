"""Numpy model of the CUDA pipeline (test infrastructure only).

Mirrors, array-wise, exactly what fm_tile.cuh / fm_tonal.cuh compute — the
in-place four-step position permutation per axis, the SE spectrum stored in
the same permuted order, the overlap-save geometry (D offsets, valid window),
the c2r packing and the Stockham stage loop with its twiddle indexing — so the
index algebra of the kernels can be checked on a CPU-only box against the
exact oracle.  It is never imported by the product package.
"""

from __future__ import annotations

import math

import numpy as np

SPLIT = {16: (4, 4), 32: (8, 4), 64: (8, 8), 128: (16, 8), 256: (16, 16)}


def smooth235(n):
    if n < 1:
        return False
    for p in (2, 3, 5):
        while n % p == 0:
            n //= p
    return n == 1


def choose_T(lr):
    T = max(2, lr + 1)
    if T % 2:
        T += 1
    while not smooth235(T // 2):
        T += 2
    return T


def radix_plan(n):
    r = []
    for p in (8, 4, 2, 3, 5):
        while n % p == 0:
            r.append(p)
            n //= p
    return r


def _fwd_axis(a, axis, P):
    """Forward four-step along `axis` with in-place position semantics (passes A+B)."""
    R1, R2 = SPLIT[P]
    a = np.moveaxis(a, axis, -1)
    sh = a.shape
    v = a.reshape(sh[:-1] + (R1, R2))          # [.., n1, n2], position n2 + R2*n1
    v = np.fft.fft(v, axis=-2)                  # pass A: DFT_R1 over n1 -> k1 (same slot)
    n2 = np.arange(R2)[None, :]
    k1 = np.arange(R1)[:, None]
    v = v * np.exp(-2j * np.pi * (n2 * k1) / P)  # twiddle W_P^{n2 k1}
    v = np.fft.fft(v, axis=-1)                  # pass B: DFT_R2 over n2 -> k2 at slot n2
    return np.moveaxis(v.reshape(sh), -1, axis)


def _inv_axis(a, axis, P):
    R1, R2 = SPLIT[P]
    a = np.moveaxis(a, axis, -1)
    sh = a.shape
    v = a.reshape(sh[:-1] + (R1, R2))
    v = np.fft.ifft(v, axis=-1) * R2            # pass B^-1 (unnormalised)
    n2 = np.arange(R2)[None, :]
    k1 = np.arange(R1)[:, None]
    v = v * np.exp(+2j * np.pi * (n2 * k1) / P)
    v = np.fft.ifft(v, axis=-2) * R1            # pass A^-1 (unnormalised)
    return np.moveaxis(v.reshape(sh), -1, axis)


def permuted_freq_check(P):
    """Position k2 + R2*k1 must hold frequency k1 + R1*k2 after _fwd_axis."""
    R1, R2 = SPLIT[P]
    x = np.random.default_rng(0).standard_normal(P) + 0j
    got = _fwd_axis(x[None, :], 1, P)[0]
    ref = np.fft.fft(x)
    for k1 in range(R1):
        for k2 in range(R2):
            assert abs(got[k2 + R2 * k1] - ref[k1 + R1 * k2]) < 1e-9
    return True


def stockham_inverse(Z, radices):
    """Per-pixel Stockham loop of fm_tonal.cuh (inverse, unnormalised)."""
    N = len(Z)
    twN = np.exp(2j * np.pi * np.arange(N) / N)
    src = np.array(Z, dtype=complex)
    Ns = 1
    for R in radices:
        dst = np.empty_like(src)
        M = N // R
        tstep = N // (Ns * R)
        for j in range(M):
            jm = j % Ns
            v = np.array([src[j + r * M] for r in range(R)])
            if Ns > 1:
                for r in range(1, R):
                    v[r] *= twN[(jm * r * tstep) % N]
            v = np.fft.ifft(v) * R
            idxD = (j // Ns) * Ns * R + jm
            for r in range(R):
                dst[idxD + r * Ns] = v[r]
        src = dst
        Ns *= R
    return src


def model_dilate(img, defined, se, se_def, se_lo, *, mode="dilate", crop=True, fill=0, P=None):
    """2-D / 1-D model of fm_execute for one image; returns (out int64, valid bool, maxdev)."""
    img = np.asarray(img, dtype=np.int64)
    two_d = img.ndim == 2
    if not two_d:
        img = img[None, :]
        defined = None if defined is None else np.asarray(defined)[None, :]
        se = np.asarray(se)[None, :]
        se_def = None if se_def is None else np.asarray(se_def)[None, :]
        se_lo = (0, se_lo[0])
    defined = np.ones(img.shape, bool) if defined is None else np.asarray(defined, bool)
    se = np.asarray(se, dtype=np.int64)
    se_def = np.ones(se.shape, bool) if se_def is None else np.asarray(se_def, bool)
    lo_y, lo_x = se_lo
    if mode == "erode":
        se = se[::-1, ::-1]
        se_def = se_def[::-1, ::-1]
        lo_y, lo_x = -(lo_y + se.shape[0] - 1), -(lo_x + se.shape[1] - 1)
    H, W = img.shape
    my, mx = se.shape
    fv = img[defined]
    img_min, img_max = int(fv.min()), int(fv.max())
    smin, smax = int(se[se_def].min()), int(se[se_def].max())
    lr = (img_max - img_min) + (smax - smin)
    T = choose_T(lr)
    N = T // 2
    if mode == "dilate":
        v_img = img - img_min
        out_sign, out_bias = 1, img_min + smin
    else:
        v_img = img_max - img
        out_sign, out_bias = -1, img_max - smin
    v_se = se - smin
    hi_y, hi_x = lo_y + my - 1, lo_x + mx - 1
    if crop:
        off_y, off_x, OH, OW = 0, 0, H, W
    else:
        off_y, off_x = (lo_y if two_d else 0), lo_x
        OH, OW = (H + my - 1 if two_d else 1), W + mx - 1
    DY, DX = (off_y - hi_y if two_d else 0), off_x - hi_x
    if P is None:
        P = next(p for p in (16, 32, 64, 128, 256) if p >= max(my if two_d else 1, mx) + 1)
    PY = P if two_d else 1
    PX = P
    QY = PY - my + 1 if two_d else 1
    QX = PX - mx + 1
    wT = np.exp(-2j * np.pi * np.arange(T) / T)
    # SE spectrum in permuted order, scaled by 1/(PY*PX*T)
    K = N + 1
    spec = np.zeros((K, PY, PX), complex)
    for k in range(K):
        plane = np.zeros((PY, PX), complex)
        for jy in range(my):
            for jx in range(mx):
                if se_def[jy, jx]:
                    plane[jy, jx] = wT[(k * v_se[jy, jx]) % T]
        s = plane
        if two_d:
            s = _fwd_axis(s, 0, PY)
        s = _fwd_axis(s, 1, PX)
        spec[k] = s / (PY * PX * T)
    chat = np.zeros((K, OH, OW), complex)
    tiles_y = -(-OH // QY)
    tiles_x = -(-OW // QX)
    for ty in range(tiles_y):
        for tx in range(tiles_x):
            tvals = np.full((PY, PX), -1, np.int64)
            for py in range(PY):
                iy = ty * QY + DY + py
                if not 0 <= iy < H:
                    continue
                for px in range(PX):
                    ix = tx * QX + DX + px
                    if 0 <= ix < W and defined[iy, ix]:
                        tvals[py, px] = v_img[iy, ix]
            for k in range(K):
                u = np.where(tvals >= 0, wT[(k * np.maximum(tvals, 0)) % T], 0)
                if two_d:
                    u = _fwd_axis(u, 0, PY)
                u = _fwd_axis(u, 1, PX)
                u = u * spec[k]
                u = _inv_axis(u, 1, PX)
                if two_d:
                    u = _inv_axis(u, 0, PY)
                for y in range(my - 1 if two_d else 0, PY):
                    oy = ty * QY + y - ((my - 1) if two_d else 0)
                    if oy >= OH:
                        continue
                    for x in range(mx - 1, PX):
                        ox = tx * QX + x - (mx - 1)
                        if ox < OW:
                            chat[k, oy, ox] = u[y, x]
    # tonal kernel
    radices = radix_plan(N)
    wTi = np.exp(2j * np.pi * np.arange(N) / T)
    out = np.zeros((OH, OW), np.int64)
    valid = np.zeros((OH, OW), bool)
    maxdev = 0.0
    for oy in range(OH):
        for ox in range(OW):
            X = chat[:, oy, ox]
            Z = np.array([(X[k] + np.conj(X[N - k])) + 1j * wTi[k] * (X[k] - np.conj(X[N - k]))
                          for k in range(N)])
            z = stockham_inverse(Z, radices)
            c = np.empty(T)
            c[0::2] = z.real
            c[1::2] = z.imag
            maxdev = max(maxdev, float(np.abs(c - np.rint(c)).max()))
            nz = np.flatnonzero(c > 0.5)
            if len(nz):
                valid[oy, ox] = True
                out[oy, ox] = out_sign * int(nz[-1]) + out_bias
            else:
                out[oy, ox] = fill
    if not two_d:
        out, valid = out[0], valid[0]
    return out, valid, maxdev


# ---------------------------------------------------------------------------
# Per-unit tonal length with the clamp bound (fm_range.cuh), modelled with
# exact integer circular counts: the tonal axis of a unit is a length-T_t
# cyclic group, so c(t) is the number of pairs whose degree is t mod T_t.

TONAL_NS = (1, 2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16, 18, 20, 24, 25, 27, 30, 32, 36, 40, 45, 48, 50,
            54, 60, 64, 72, 75, 80, 81, 90, 96, 100, 108, 120, 125, 128, 135, 144, 150, 160)


def bound_taps(se, se_def, cap=128):
    """Tap order of fm_abi.cu: highest value first, ties by a multiplicative hash of the index."""
    my, mx = se.shape
    smax = int(se[se_def].max())
    cand = []
    for py in range(my):
        for px in range(mx):
            i = py * mx + px
            if se_def[py, px]:
                h = (i * 2654435761) & 0xFFFFFFFF
                cand.append((((smax - int(se[py, px])) << 32) | h, (my - 1 - py, mx - 1 - px)))
    cand.sort()
    return [c[1] for c in cand[:cap]]


def model_clamped_units(img, defined, se, se_def, se_lo, *, mode="dilate", crop=True, fill=0, P=None,
                        cap=128):
    """Per-unit (anchor, T_t) of fm_range.cuh and the exact result through circular counts.

    Returns (out, valid, mean_planes) for one 2-D image (1-D: pass shape (1, W) arrays)."""
    img = np.asarray(img, dtype=np.int64)
    defined = np.ones(img.shape, bool) if defined is None else np.asarray(defined, bool)
    se = np.asarray(se, dtype=np.int64)
    se_def = np.ones(se.shape, bool) if se_def is None else np.asarray(se_def, bool)
    lo_y, lo_x = se_lo
    if mode == "erode":
        se, se_def = se[::-1, ::-1], se_def[::-1, ::-1]
        lo_y, lo_x = -(lo_y + se.shape[0] - 1), -(lo_x + se.shape[1] - 1)
    H, W = img.shape
    my, mx = se.shape
    fv = img[defined]
    img_min, img_max = int(fv.min()), int(fv.max())
    smin, smax = int(se[se_def].min()), int(se[se_def].max())
    lr_se = smax - smin
    N_glob = choose_T((img_max - img_min) + lr_se) // 2
    ladder = [n for n in TONAL_NS if n < N_glob] + [N_glob]
    enc_sign, enc_bias = (1, -img_min) if mode == "dilate" else (-1, img_max)
    out_sign = 1 if mode == "dilate" else -1
    vg = np.where(defined, enc_sign * img + enc_bias, -1)
    bp = se - smin
    hi_y, hi_x = lo_y + my - 1, lo_x + mx - 1
    if crop:
        off_y, off_x, OH, OW = 0, 0, H, W
    else:
        off_y, off_x, OH, OW = lo_y, lo_x, H + my - 1, W + mx - 1
    DY, DX = off_y - hi_y, off_x - hi_x
    if P is None:
        P = next(p for p in (16, 32, 64, 128, 256) if p >= max(my, mx) + 1)
    PY = P if H > 1 or my > 1 else 1
    QY, QX = PY - my + 1, P - mx + 1
    taps = bound_taps(se, se_def, cap)
    out = np.zeros((OH, OW), np.int64)
    valid = np.zeros((OH, OW), bool)
    planes = []
    for ty in range(-(-OH // QY)):
        for tx in range(-(-OW // QX)):
            y0, x0 = ty * QY + DY, tx * QX + DX
            win = np.full((PY, P), -1, np.int64)
            for r in range(PY):
                for c in range(P):
                    iy, ix = y0 + r, x0 + c
                    if 0 <= iy < H and 0 <= ix < W:
                        win[r, c] = vg[iy, ix]
            vals = win[win >= 0]
            if vals.size == 0:
                lo = hi = 0
                any_ = False
            else:
                lo, hi, any_ = int(vals.min()), int(vals.max()), True
            ny, nx = min(QY, OH - ty * QY), min(QX, OW - tx * QX)
            c = lo
            if any_:
                D = None
                for jy in range(ny):
                    for jx in range(nx):
                        g = -(1 << 40)
                        for (dy, dx) in taps:
                            s = win[jy + dy, jx + dx]
                            g = max(g, (s if s >= 0 else -32768) + int(bp[my - 1 - dy, mx - 1 - dx]))
                        D = g if D is None else min(D, g)
                # fm_range.cuh reports the ladder breakpoint level of the minimum
                # (hi + 2 lr_se - 2N + 1 for the smallest N whose level is <= D)
                if D is not None:
                    lev = next((hi + 2 * lr_se - 2 * n + 1 for n in ladder if hi + 2 * lr_se - 2 * n + 1 <= D), None)
                    D = lev if lev is not None and lev > lo + lr_se else None
                if D is not None and D - lr_se > c:
                    c = min(D - lr_se, hi)
            lr = (hi - c) + lr_se if any_ else lr_se
            N = next((n for n in ladder if 2 * n >= lr + 1), ladder[-1])
            T = 2 * N
            planes.append(N + 1)
            anchor = enc_sign * (c - enc_bias)
            for jy in range(ny):
                for jx in range(nx):
                    cnt = np.zeros(T, np.int64)
                    for py in range(my):
                        for px in range(mx):
                            if not se_def[py, px]:
                                continue
                            s = win[jy + (my - 1 - py), jx + (mx - 1 - px)]
                            if s >= 0:
                                cnt[(max(s - c, 0) + bp[py, px]) % T] += 1
                    nz = np.flatnonzero(cnt)
                    oy, ox = ty * QY + jy, tx * QX + jx
                    if len(nz):
                        valid[oy, ox] = True
                        out[oy, ox] = out_sign * (int(nz[-1]) + smin) + anchor
                    else:
                        out[oy, ox] = fill
    return out, valid, float(np.mean(planes))
