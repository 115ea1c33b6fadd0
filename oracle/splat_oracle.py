"""ORACLE — test infrastructure only (see oracle/__init__.py).

float64 numpy restatement of the reference hot path.  Citations are
``path:line`` relative to /root/reference/pkg/src/splatstream/.

Inputs are duck-typed: a camera is anything with ``width, height, fx, fy,
cx, cy, rotation (3,3), translation (3,)``; splat arrays are passed as
explicit numpy arrays (means, quats, scales, opacities, colors) so this
module imports nothing from the product package.
"""

from __future__ import annotations

import ctypes
import math
import os
from pathlib import Path

import numpy as np

NEAR_PLANE = 0.01          # raster.py:31
COV2D_DILATION = 0.3       # raster.py:34
ALPHA_MAX = 0.999          # _kernels.py:15
T_MIN = 1e-4               # _kernels.py:16
MAHA_MAX = 64.0            # _kernels.py:17
SCALE_FLOOR = 1e-6         # core.py:15
SSIM_C1 = 0.01 ** 2        # loss.py:14
SSIM_C2 = 0.03 ** 2        # loss.py:15
TILE = 16                  # build's tile edge (a-4); not a reference constant
RANK_BITS = 21             # key = tile << 21 | depth rank
# Alpha floor of the build's binning (libswings ss_set_alpha_floor, default
# -28): a (splat, tile) pair is emitted only where alpha G >= 2^-28 can hold
# at some pixel of the tile, i.e. m <= 2 ln(alpha / 2^-28) as well as
# m <= 64.  Skipped contributions are below 2^-28 each: the image moves by
# at most ~2 |S| 2^-28 (|S| = skipped entries of a pixel), far inside the
# north star's 1e-4.  None = the reference's maha <= 64 rule only.
ALPHA_FLOOR_LOG2 = -28
TWO_LN2 = 1.3862943611198906
PARAM_GROUPS = ("mean", "quat", "log_scale", "opacity_logit", "color")  # train.py:39

_HERE = Path(__file__).resolve().parent
_LIB = None


def _lib():
    """The compiled C restatement of the pixel loops (oracle/blend.c)."""
    global _LIB
    if _LIB is None:
        path = _HERE / "_build" / "liboracle_blend.so"
        if not path.exists():
            build_oracle()
        lib = ctypes.CDLL(str(path))
        P = ctypes.c_void_p
        I = ctypes.c_int64
        lib.oracle_blend_forward.argtypes = [P, I, P, P, P, P, P, P, P, P, I, I, P, ctypes.c_int]
        lib.oracle_blend_backward.argtypes = [P, I, P, P, P, P, P, P, P, P, I, I, P, P, P, P, P, I,
                                              ctypes.c_int]
        lib.oracle_blend_forward_tiled.argtypes = [P, P, I, P, P, P, P, P, P, P, P, I, I, P, P, P, P,
                                                   ctypes.c_int]
        lib.oracle_blend_backward_tiled.argtypes = [P, P, I, P, P, P, P, P, P, P, P, I, I, P, P, P,
                                                    P, P, I, ctypes.c_int]
        _LIB = lib
    return _LIB


def build_oracle() -> Path:
    """Compile oracle/blend.c with the recipe in oracle/Makefile."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _HERE / "_build" / "liboracle_blend.so"


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


# --------------------------------------------------------------------------
# core.py restatements
# --------------------------------------------------------------------------

def quat_to_rotmat(q):
    """core.py:231-251 — rotation matrix of (w, x, y, z) quaternions (N,4)->(N,3,3)."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    r = np.empty((len(q), 3, 3))
    r[:, 0, 0] = 1 - 2 * (y * y + z * z)
    r[:, 0, 1] = 2 * (x * y - w * z)
    r[:, 0, 2] = 2 * (x * z + w * y)
    r[:, 1, 0] = 2 * (x * y + w * z)
    r[:, 1, 1] = 1 - 2 * (x * x + z * z)
    r[:, 1, 2] = 2 * (y * z - w * x)
    r[:, 2, 0] = 2 * (x * z - w * y)
    r[:, 2, 1] = 2 * (y * z + w * x)
    r[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def sigmoid(x):
    """train.py:134-135."""
    return 1.0 / (1.0 + np.exp(-x))


def logit(p):
    """train.py:129-131 (clipped to [1e-9, 1-1e-9])."""
    p = np.clip(p, 1e-9, 1.0 - 1e-9)
    return np.log(p / (1.0 - p))


def active_rows(starts, expires, frame):
    """Active-set compaction, core.py:280-282 + train.py:347-350, 380-386.

    ``starts``/``expires`` are per candidate row in the reference's
    concatenation order (optimizable generations in ``state.slices`` order,
    then matured generations in archive order).  Returns the indices of the
    rows with ``start <= frame < expire``, ascending (= concat order).
    """
    starts = np.asarray(starts)
    expires = np.asarray(expires)
    return np.nonzero((starts <= frame) & (frame < expires))[0]


# --------------------------------------------------------------------------
# raster.py restatements
# --------------------------------------------------------------------------

def project_arrays(cam, means, quats, scales, opacities, colors):
    """raster.py:76-173 — EWA projection, 3-sigma cull, dilation, conic, 8-sigma bbox,
    global (z, src) order.  Returns None when nothing survives."""
    n = len(means)
    if n == 0:
        return None
    rot_wc = np.asarray(cam.rotation, dtype=np.float64)
    t = means @ rot_wc.T + np.asarray(cam.translation, dtype=np.float64)   # raster.py:86
    z = t[:, 2]
    in_front = z > NEAR_PLANE                                                # raster.py:88
    with np.errstate(divide="ignore", invalid="ignore"):
        ux = cam.fx * t[:, 0] / z + cam.cx                                   # raster.py:91-92
        uy = cam.fy * t[:, 1] / z + cam.cy
    qnorm = np.linalg.norm(quats, axis=1)                                    # raster.py:94-95
    qn = quats / np.maximum(qnorm, 1e-12)[:, None]
    rot = quat_to_rotmat(qn)
    m3 = rot * scales[:, None, :]                                            # raster.py:97-98
    sigma = m3 @ np.transpose(m3, (0, 2, 1))
    jac = np.zeros((n, 2, 3))                                                # raster.py:101-106
    with np.errstate(divide="ignore", invalid="ignore"):
        jac[:, 0, 0] = cam.fx / z
        jac[:, 0, 2] = -cam.fx * t[:, 0] / (z * z)
        jac[:, 1, 1] = cam.fy / z
        jac[:, 1, 2] = -cam.fy * t[:, 1] / (z * z)
    mproj = jac @ rot_wc                                                     # raster.py:107
    cov2d = np.einsum("nab,nbc,ndc->nad", mproj, sigma, mproj)               # raster.py:108
    a_raw, b_raw, c_raw = cov2d[:, 0, 0], cov2d[:, 0, 1], cov2d[:, 1, 1]
    mid = 0.5 * (a_raw + c_raw)                                              # raster.py:114-122
    disc = np.sqrt(np.maximum(mid * mid - (a_raw * c_raw - b_raw * b_raw), 0.0))
    r3 = 3.0 * np.sqrt(np.maximum(mid + disc, 0.0))
    on_image = ((ux + r3 >= 0.0) & (ux - r3 <= cam.width - 1.0)
                & (uy + r3 >= 0.0) & (uy - r3 <= cam.height - 1.0))
    src = np.nonzero(in_front & on_image)[0]                                 # raster.py:123-124
    if len(src) == 0:
        return None
    t, z = t[src], z[src]
    mean2d = np.column_stack([ux[src], uy[src]])
    a_raw, b_raw, c_raw = a_raw[src], b_raw[src], c_raw[src]
    ad = a_raw + COV2D_DILATION                                              # raster.py:139-142
    cd = c_raw + COV2D_DILATION
    det = ad * cd - b_raw * b_raw
    inv2d = np.column_stack([cd / det, -b_raw / det, ad / det])
    mid_d = 0.5 * (ad + cd)                                                  # raster.py:144-150
    disc_d = np.sqrt(np.maximum(mid_d * mid_d - det, 0.0))
    r8 = 8.0 * np.sqrt(mid_d + disc_d)
    x0 = np.maximum(np.ceil(mean2d[:, 0] - r8), 0.0).astype(np.int64)
    x1 = np.minimum(np.floor(mean2d[:, 0] + r8) + 1.0, cam.width).astype(np.int64)
    y0 = np.maximum(np.ceil(mean2d[:, 1] - r8), 0.0).astype(np.int64)
    y1 = np.minimum(np.floor(mean2d[:, 1] + r8) + 1.0, cam.height).astype(np.int64)
    order = np.lexsort((src, z)).astype(np.int64)                            # raster.py:153
    return {
        "src": src, "t": t, "z": z, "mean2d": np.ascontiguousarray(mean2d),
        "cov_raw": (a_raw, b_raw, c_raw), "dilated": (ad, b_raw, cd, det),
        "inv2d": np.ascontiguousarray(inv2d), "qn": qn[src], "qnorm": qnorm[src],
        "rot": rot[src], "m3": m3[src], "sigma": sigma[src], "mproj": mproj[src],
        "bbox": (x0, x1, y0, y1), "order": order,
        "alpha": np.ascontiguousarray(opacities[src]),
        "color": np.ascontiguousarray(colors[src]),
        "scales": scales[src],
    }


def _blend_args(cache):
    x0, x1, y0, y1 = (np.ascontiguousarray(b, dtype=np.int64) for b in cache["bbox"])
    return (cache["mean2d"], cache["inv2d"], cache["alpha"], np.ascontiguousarray(cache["color"]),
            x0, x1, y0, y1)


def blend_forward(cache, height, width, nthreads=1):
    """_kernels.py:20-53 via oracle/blend.c (global order, reference loop)."""
    img = np.zeros((height, width, 3))
    m2, inv, al, col, x0, x1, y0, y1 = _blend_args(cache)
    order = np.ascontiguousarray(cache["order"], dtype=np.int64)
    _lib().oracle_blend_forward(_p(order), len(order), _p(m2), _p(inv), _p(al), _p(col), _p(x0),
                                _p(x1), _p(y0), _p(y1), height, width, _p(img), nthreads)
    return img


def blend_backward(cache, height, width, grad_img, nthreads=1):
    """_kernels.py:56-130 via oracle/blend.c; returns (g_mean2d, g_inv2d, g_alpha, g_color)."""
    p = len(cache["src"])
    g_mean2d, g_inv2d = np.zeros((p, 2)), np.zeros((p, 3))
    g_alpha, g_color = np.zeros(p), np.zeros((p, 3))
    m2, inv, al, col, x0, x1, y0, y1 = _blend_args(cache)
    order = np.ascontiguousarray(cache["order"], dtype=np.int64)
    gi = np.ascontiguousarray(grad_img, dtype=np.float64)
    _lib().oracle_blend_backward(_p(order), len(order), _p(m2), _p(inv), _p(al), _p(col), _p(x0),
                                 _p(x1), _p(y0), _p(y1), height, width, _p(gi), _p(g_mean2d),
                                 _p(g_inv2d), _p(g_alpha), _p(g_color), p, nthreads)
    return g_mean2d, g_inv2d, g_alpha, g_color


def render_arrays(cam, means, quats, scales, opacities, colors, nthreads=1, tiled=False):
    """raster.py:194-204 — (H, W, 3) float64 linear RGB."""
    cache = project_arrays(cam, means, quats, scales, opacities, colors)
    if cache is None:
        return np.zeros((cam.height, cam.width, 3))
    if tiled:
        return blend_forward_tiled(cache, cam.height, cam.width, nthreads)["image"]
    return blend_forward(cache, cam.height, cam.width, nthreads)


def projection_backward(cam, cache, n, g_mean2d, g_inv2d, g_alpha, g_color, trainable=None):
    """raster.py:249-348 — chain 2D gradients to optimization-space gradients
    aligned with the input rows (mean, log_scale, raw quat, opacity logit, colour)."""
    grads = {
        "mean": np.zeros((n, 3)), "log_scale": np.zeros((n, 3)), "quat": np.zeros((n, 4)),
        "opacity_logit": np.zeros((n,)), "color": np.zeros((n, 3)),
    }
    src, t, z = cache["src"], cache["t"], cache["z"]
    ad, b, cd, det = cache["dilated"]
    sigma, m3, rot, qn, qnorm, mproj = (cache[k] for k in ("sigma", "m3", "rot", "qn", "qnorm", "mproj"))
    fx, fy = cam.fx, cam.fy
    det2 = det * det                                                         # raster.py:262-266
    gia, gib, gic = g_inv2d[:, 0], g_inv2d[:, 1], g_inv2d[:, 2]
    g_a = (gia * (-cd * cd) + gib * (b * cd) + gic * (-b * b)) / det2
    g_b = (gia * (2.0 * b * cd) + gib * (-det - 2.0 * b * b) + gic * (2.0 * ad * b)) / det2
    g_c = (gia * (-b * b) + gib * (ad * b) + gic * (-ad * ad)) / det2
    m0, m1 = mproj[:, 0, :], mproj[:, 1, :]                                  # raster.py:269-280
    sm0 = np.einsum("pij,pj->pi", sigma, m0)
    sm1 = np.einsum("pij,pj->pi", sigma, m1)
    gm = np.empty_like(mproj)
    gm[:, 0, :] = 2.0 * g_a[:, None] * sm0 + g_b[:, None] * sm1
    gm[:, 1, :] = g_b[:, None] * sm0 + 2.0 * g_c[:, None] * sm1
    g_sigma = (g_a[:, None, None] * np.einsum("pi,pj->pij", m0, m0)
               + g_b[:, None, None] * np.einsum("pi,pj->pij", m0, m1)
               + g_c[:, None, None] * np.einsum("pi,pj->pij", m1, m1))
    rot_wc = np.asarray(cam.rotation, dtype=np.float64)
    gj = gm @ rot_wc.T                                                       # raster.py:283-300
    x_c, y_c = t[:, 0], t[:, 1]
    z2 = z * z
    z3 = z2 * z
    gt = np.zeros((len(src), 3))
    gt[:, 0] = gj[:, 0, 2] * (-fx / z2)
    gt[:, 1] = gj[:, 1, 2] * (-fy / z2)
    gt[:, 2] = (gj[:, 0, 0] * (-fx / z2) + gj[:, 1, 1] * (-fy / z2)
                + gj[:, 0, 2] * (2.0 * fx * x_c / z3) + gj[:, 1, 2] * (2.0 * fy * y_c / z3))
    gt[:, 0] += g_mean2d[:, 0] * fx / z
    gt[:, 1] += g_mean2d[:, 1] * fy / z
    gt[:, 2] += -g_mean2d[:, 0] * fx * x_c / z2 - g_mean2d[:, 1] * fy * y_c / z2
    g_mean = gt @ rot_wc
    gm3 = (g_sigma + np.transpose(g_sigma, (0, 2, 1))) @ m3                  # raster.py:303-306
    g_scale = np.einsum("pik,pik->pk", gm3, rot)
    scales = cache["scales"]
    g_log_scale = g_scale * scales
    gr = gm3 * scales[:, None, :]                                            # raster.py:308-334
    w, x, y, zz = qn[:, 0], qn[:, 1], qn[:, 2], qn[:, 3]
    zero = np.zeros_like(w)
    dr = np.empty((len(src), 4, 3, 3))
    dr[:, 0] = 2.0 * np.stack([np.stack([zero, -zz, y], -1), np.stack([zz, zero, -x], -1),
                               np.stack([-y, x, zero], -1)], 1)
    dr[:, 1] = 2.0 * np.stack([np.stack([zero, y, zz], -1), np.stack([y, -2 * x, -w], -1),
                               np.stack([zz, w, -2 * x], -1)], 1)
    dr[:, 2] = 2.0 * np.stack([np.stack([-2 * y, x, w], -1), np.stack([x, zero, zz], -1),
                               np.stack([-w, zz, -2 * y], -1)], 1)
    dr[:, 3] = 2.0 * np.stack([np.stack([-2 * zz, -w, x], -1), np.stack([w, -2 * zz, y], -1),
                               np.stack([x, y, zero], -1)], 1)
    g_qn = np.einsum("pik,pqik->pq", gr, dr)
    g_quat = (g_qn - qn * np.sum(qn * g_qn, axis=1, keepdims=True)) / qnorm[:, None]
    alpha = cache["alpha"]
    g_logit = g_alpha * alpha * (1.0 - alpha)                                # raster.py:336-337
    grads["mean"][src] = g_mean                                              # raster.py:339-347
    grads["log_scale"][src] = g_log_scale
    grads["quat"][src] = g_quat
    grads["opacity_logit"][src] = g_logit
    grads["color"][src] = g_color
    if trainable is not None:
        mask = ~np.asarray(trainable, dtype=bool)
        for v in grads.values():
            v[mask] = 0.0
    return grads


def render_arrays_backward(cam, means, quats, scales, opacities, colors, grad_image,
                           trainable=None, nthreads=1, tiled=False):
    """raster.py:207-348."""
    n = len(means)
    grad_image = np.ascontiguousarray(grad_image, dtype=np.float64)
    cache = project_arrays(cam, means, quats, scales, opacities, colors)
    if cache is None:
        return {"mean": np.zeros((n, 3)), "log_scale": np.zeros((n, 3)), "quat": np.zeros((n, 4)),
                "opacity_logit": np.zeros((n,)), "color": np.zeros((n, 3))}
    if tiled:
        bins = tile_bins(cache, cam.width, cam.height, floor_log2=None)
        g2d = blend_backward_tiled(cache, bins, cam.height, cam.width, grad_image, nthreads)
    else:
        g2d = blend_backward(cache, cam.height, cam.width, grad_image, nthreads)
    return projection_backward(cam, cache, n, *g2d, trainable=trainable)


# --------------------------------------------------------------------------
# a-4: tile binning restated (build design; reproduces the reference order)
# --------------------------------------------------------------------------

def tile_bins(cache, width, height, tile=TILE, exact=True, floor_log2=ALPHA_FLOOR_LOG2):
    """SURVEY.md §8 a-4.  For each kept splat i (index into the kept subset)
    with depth rank r_i under the reference's global (z, src) order
    (raster.py:153), emit one key ``tile_id << 21 | r_i`` per 16x16 tile
    overlapping its half-open pixel bbox [x0,x1)x[y0,y1) (raster.py:144-150)
    -- with ``exact``, only tiles the maha <= 64 ellipse reaches
    (tile_keep_mask; dropped tiles hold no pixel the reference blends) and,
    with ``floor_log2`` (the library default), only those where
    alpha G >= 2^floor_log2 can hold (None: the reference rule alone; the
    per-pixel oracles on those bins are then the reference's exact walk) --
    sort keys ascending; a tile's range is the run of its tile id.

    Returns dict(keys (K,) uint64 sorted, vals (K,) int64 kept-subset index,
    ranges (T,2) int64 [start,end), tiles_x, tiles_y, K).
    """
    order = cache["order"]
    p = len(order)
    rank = np.empty(p, dtype=np.int64)
    rank[order] = np.arange(p, dtype=np.int64)
    x0, x1, y0, y1 = cache["bbox"]
    tiles_x = (width + tile - 1) // tile
    tiles_y = (height + tile - 1) // tile
    nonempty = (x1 > x0) & (y1 > y0)
    tx0 = np.where(nonempty, x0 // tile, 0)
    tx1 = np.where(nonempty, (x1 - 1) // tile + 1, 0)
    ty0 = np.where(nonempty, y0 // tile, 0)
    ty1 = np.where(nonempty, (y1 - 1) // tile + 1, 0)
    counts = (tx1 - tx0) * (ty1 - ty0)
    total = int(counts.sum())
    owner = np.repeat(np.arange(p, dtype=np.int64), counts)
    start = np.repeat(np.cumsum(counts) - counts, counts)
    local = np.arange(total, dtype=np.int64) - start
    w = np.repeat(tx1 - tx0, counts)
    tx = np.repeat(tx0, counts) + local % np.maximum(w, 1)
    ty = np.repeat(ty0, counts) + local // np.maximum(w, 1)
    if exact and total:
        keep = tile_keep_mask(cache, owner, tx, ty, tile, floor_log2)
        owner, tx, ty = owner[keep], tx[keep], ty[keep]
        total = int(keep.sum())
    tile_id = ty * tiles_x + tx
    keys = (tile_id.astype(np.uint64) << np.uint64(RANK_BITS)) | rank[owner].astype(np.uint64)
    srt = np.argsort(keys, kind="stable")
    keys = keys[srt]
    vals = owner[srt]
    n_tiles = tiles_x * tiles_y
    tid_sorted = (keys >> np.uint64(RANK_BITS)).astype(np.int64)
    ranges = np.zeros((n_tiles, 2), dtype=np.int64)
    ranges[:, 0] = np.searchsorted(tid_sorted, np.arange(n_tiles), side="left")
    ranges[:, 1] = np.searchsorted(tid_sorted, np.arange(n_tiles), side="right")
    return {"keys": keys, "vals": vals, "ranges": ranges, "tiles_x": tiles_x,
            "tiles_y": tiles_y, "K": total}


def blend_forward_tiled(cache, height, width, nthreads=1, bins=None):
    """Tiled restatement of _kernels.py:20-53 (same per-pixel sequence).  Also
    returns per-pixel walked entries, contributors and final T, and K_used
    (SURVEY.md §8 notation)."""
    if bins is None:
        bins = tile_bins(cache, width, height, floor_log2=None)  # the reference's exact walk
    img = np.zeros((height, width, 3))
    walked = np.zeros(height * width, dtype=np.int64)
    contrib = np.zeros(height * width, dtype=np.int64)
    t_final = np.zeros(height * width)
    m2, inv, al, col, x0, x1, y0, y1 = _blend_args(cache)
    ranges = np.ascontiguousarray(bins["ranges"], dtype=np.int64)
    vals = np.ascontiguousarray(bins["vals"], dtype=np.int64)
    _lib().oracle_blend_forward_tiled(_p(ranges), _p(vals), bins["tiles_x"], _p(m2), _p(inv), _p(al),
                                      _p(col), _p(x0), _p(x1), _p(y0), _p(y1), height, width,
                                      _p(img), _p(walked), _p(contrib), _p(t_final), nthreads)
    tx = np.arange(width) // TILE
    ty = np.arange(height) // TILE
    tile_of_px = (ty[:, None] * bins["tiles_x"] + tx[None, :]).reshape(-1)
    per_tile_max = np.zeros(bins["tiles_x"] * bins["tiles_y"], dtype=np.int64)
    np.maximum.at(per_tile_max, tile_of_px, walked)
    return {"image": img, "walked": walked.reshape(height, width),
            "contrib": contrib.reshape(height, width), "t_final": t_final.reshape(height, width),
            "K": bins["K"], "K_used": int(per_tile_max.sum()), "bins": bins}


def blend_backward_tiled(cache, bins, height, width, grad_img, nthreads=1):
    p = len(cache["src"])
    g_mean2d, g_inv2d = np.zeros((p, 2)), np.zeros((p, 3))
    g_alpha, g_color = np.zeros(p), np.zeros((p, 3))
    m2, inv, al, col, x0, x1, y0, y1 = _blend_args(cache)
    ranges = np.ascontiguousarray(bins["ranges"], dtype=np.int64)
    vals = np.ascontiguousarray(bins["vals"], dtype=np.int64)
    gi = np.ascontiguousarray(grad_img, dtype=np.float64)
    _lib().oracle_blend_backward_tiled(_p(ranges), _p(vals), bins["tiles_x"], _p(m2), _p(inv),
                                       _p(al), _p(col), _p(x0), _p(x1), _p(y0), _p(y1), height,
                                       width, _p(gi), _p(g_mean2d), _p(g_inv2d), _p(g_alpha),
                                       _p(g_color), p, nthreads)
    return g_mean2d, g_inv2d, g_alpha, g_color


# --------------------------------------------------------------------------
# loss.py restatements
# --------------------------------------------------------------------------

def gaussian_window(size=11, sigma=1.5):
    """loss.py:20-23."""
    x = np.arange(size) - (size - 1) / 2.0
    w = np.exp(-(x ** 2) / (2.0 * sigma ** 2))
    return w / w.sum()


_WIN = gaussian_window()


def blur(img):
    """loss.py:29-32: separable 11-tap Gaussian, zero padding, axis 0 then axis 1.
    Restated as explicit shifted sums (scipy.ndimage.convolve1d mode='constant')."""
    def along(a, axis):
        out = np.zeros_like(a)
        n = a.shape[axis]
        r = len(_WIN) // 2
        for k, wk in enumerate(_WIN):
            off = k - r   # out[i] += w[k] * a[i + off]
            lo, hi = max(0, -off), min(n, n - off)
            if hi <= lo:
                continue
            src = [slice(None)] * a.ndim
            dst = [slice(None)] * a.ndim
            dst[axis] = slice(lo, hi)
            src[axis] = slice(lo + off, hi + off)
            out[tuple(dst)] += wk * a[tuple(src)]
        return out
    return along(along(img, 0), 1)


def ssim_with_gradient(x, y):
    """loss.py:35-60."""
    mu_x, mu_y = blur(x), blur(y)
    mxx, mxy, myy = blur(x * x), blur(x * y), blur(y * y)
    sig_x = mxx - mu_x * mu_x
    sig_y = myy - mu_y * mu_y
    sig_xy = mxy - mu_x * mu_y
    a1 = 2.0 * mu_x * mu_y + SSIM_C1
    a2 = 2.0 * sig_xy + SSIM_C2
    b1 = mu_x * mu_x + mu_y * mu_y + SSIM_C1
    b2 = sig_x + sig_y + SSIM_C2
    denom = b1 * b2
    s = (a1 * a2) / denom
    value = float(np.mean(s))
    ds_dmu = (2.0 * mu_y * (a2 - a1) - 2.0 * mu_x * s * (b2 - b1)) / denom
    ds_dmxx = -s / b2
    ds_dmxy = 2.0 * a1 / denom
    grad = (blur(ds_dmu) + 2.0 * x * blur(ds_dmxx) + y * blur(ds_dmxy)) / s.size
    return value, grad


def loss(pred, gt, opt_opacities, opt_scales, ssim_weight=0.2, opacity_reg=2e-2,
         scale_reg=1e-2):
    """loss.py:73-118.  Returns (breakdown dict, grad_image, reg_grads dict)."""
    diff = pred - gt
    l1 = float(np.mean(np.abs(diff)))
    ssim_val, ssim_grad = ssim_with_gradient(pred, gt)
    photometric = (1.0 - ssim_weight) * l1 + ssim_weight * (1.0 - ssim_val)
    grad_image = (1.0 - ssim_weight) * np.sign(diff) / diff.size - ssim_weight * ssim_grad
    n = len(opt_opacities)
    reg = {"opacity_logit": np.zeros((n,)), "log_scale": np.zeros((n, 3))}
    opacity_term = scale_term = 0.0
    if n > 0:
        opacity_term = opacity_reg * float(np.mean(opt_opacities))
        scale_term = scale_reg * float(np.mean(np.sum(opt_scales, axis=1)))
        reg["opacity_logit"] = opacity_reg * opt_opacities * (1.0 - opt_opacities) / n
        reg["log_scale"] = scale_reg * opt_scales / n
    total = photometric + opacity_term + scale_term
    br = {"total": total, "l1": l1, "ssim": ssim_val, "photometric": photometric,
          "opacity_term": opacity_term, "scale_term": scale_term}
    return br, grad_image, reg


def srgb_to_linear(y):
    """raster.py:416-418."""
    y = np.clip(y, 0.0, 1.0)
    return np.where(y <= 0.04045, y / 12.92, np.power((y + 0.055) / 1.055, 2.4))


def linear_to_srgb(x):
    """raster.py:411-413."""
    x = np.clip(x, 0.0, 1.0)
    return np.where(x <= 0.0031308, 12.92 * x, 1.055 * np.power(x, 1.0 / 2.4) - 0.055)


def u8_from_linear(img):
    """write_png's quantisation, raster.py:421-425 (without the PNG container)."""
    return np.rint(linear_to_srgb(img) * 255.0).astype(np.uint8)


def linear_from_u8(u8):
    """read_png's decode, raster.py:428-432 (without the PNG container)."""
    return srgb_to_linear(np.asarray(u8, dtype=np.float64) / 255.0)


# --------------------------------------------------------------------------
# train.py restatements (optimizer, SGLD with injected eta, relocation with
# injected uniforms)
# --------------------------------------------------------------------------

def group_lr(cfg, group):
    """train.py:97-104."""
    return {"mean": cfg["lr_mean"], "quat": cfg["lr_quat"], "log_scale": cfg["lr_log_scale"],
            "opacity_logit": cfg["lr_opacity_logit"], "color": cfg["lr_color"]}[group]


DEFAULT_CFG = dict(lr_mean=1.6e-4, lr_quat=1e-3, lr_log_scale=5e-3, lr_opacity_logit=5e-2,
                   lr_color=2.5e-3, adam_beta1=0.9, adam_beta2=0.999, adam_eps=1e-15,
                   optimizer="adam", noise_lr=5e4, noise_gate_center=0.005,
                   noise_gate_sharpness=100.0, gradient_scale_decay=0.5,
                   dead_opacity_threshold=0.005, opacity_reg=2e-2, scale_reg=1e-2,
                   ssim_weight=0.2)


def optimizer_step(params, m, v, t, grads, cfg=DEFAULT_CFG):
    """train.py:321-344 — one step of the generation's optimizer, in place.
    ``t`` is the generation's adam_t BEFORE the step; returns the new t."""
    if cfg["optimizer"] == "sgd":
        for k in PARAM_GROUPS:
            params[k] -= group_lr(cfg, k) * grads[k]
    else:
        t += 1
        b1, b2, eps = cfg["adam_beta1"], cfg["adam_beta2"], cfg["adam_eps"]
        bc1 = 1.0 - b1 ** t
        bc2 = 1.0 - b2 ** t
        for k in PARAM_GROUPS:
            g = grads[k]
            m[k] *= b1
            m[k] += (1.0 - b1) * g
            v[k] *= b2
            v[k] += (1.0 - b2) * g * g
            step = (m[k] / bc1) / (np.sqrt(v[k] / bc2) + eps)
            params[k] -= group_lr(cfg, k) * step
    q = params["quat"]
    q /= np.maximum(np.linalg.norm(q, axis=1, keepdims=True), 1e-12)
    np.clip(params["color"], 0.0, 1.0, out=params["color"])
    np.maximum(params["log_scale"], math.log(SCALE_FLOOR), out=params["log_scale"])
    return t


def sgld_perturb(params_list, current_mean_lr, noise_lr, etas, gate_center=0.005,
                 gate_sharpness=100.0):
    """train.py:246-264 with eta injected (one (n,3) array per generation, in the
    order the reference draws them)."""
    for p, eta in zip(params_list, etas):
        alpha = sigmoid(p["opacity_logit"])
        gate = sigmoid(-gate_sharpness * (alpha - gate_center))
        rot = quat_to_rotmat(p["quat"])
        lmat = rot * np.exp(p["log_scale"])[:, None, :]
        step = np.einsum("nij,nj->ni", lmat, eta)
        p["mean"] += (noise_lr * current_mean_lr) * gate[:, None] * step


def relocation_targets(alpha, threshold, uniforms):
    """train.py:279-294 with numpy Generator.choice's p-sampling restated:
    cdf = cumsum(p); cdf /= cdf[-1]; idx = searchsorted(cdf, u, 'right')."""
    dead = np.nonzero(alpha < threshold)[0]
    alive = np.nonzero(alpha >= threshold)[0]
    if len(dead) == 0 or len(alive) == 0:
        return dead, alive, np.zeros(0, dtype=np.int64)
    probs = alpha[alive] / alpha[alive].sum()
    cdf = probs.cumsum()
    cdf /= cdf[-1]
    idx = cdf.searchsorted(np.asarray(uniforms[: len(dead)]), side="right")
    return dead, alive, alive[idx]


def relocate(params_list, m_list, v_list, threshold, uniforms):
    """train.py:267-318 with the choice() uniforms injected.  Returns #relocated."""
    if not params_list:
        return 0
    counts = [len(p["mean"]) for p in params_list]
    offsets = np.cumsum([0] + counts)
    alpha = np.concatenate([sigmoid(p["opacity_logit"]) for p in params_list])
    dead, alive, targets = relocation_targets(alpha, threshold, uniforms)
    if len(dead) == 0 or len(alive) == 0:
        return 0

    def locate(flat):
        gi = int(np.searchsorted(offsets, flat, side="right") - 1)
        return gi, int(flat - offsets[gi])

    by_target = {}
    for d, t in zip(dead, targets):
        by_target.setdefault(int(t), []).append(int(d))
    for t, clones in by_target.items():
        nc = len(clones)
        tg, tr = locate(t)
        tp = params_list[tg]
        o_t = float(sigmoid(tp["opacity_logit"][tr]))
        o_new = 1.0 - (1.0 - o_t) ** (1.0 / (nc + 1))
        new_logit = float(logit(o_new))
        tp["opacity_logit"][tr] = new_logit
        clone_ls = tp["log_scale"][tr] - 0.5 * math.log(nc + 1)
        for d in clones:
            dg, dr = locate(d)
            dp = params_list[dg]
            dp["mean"][dr] = tp["mean"][tr]
            dp["quat"][dr] = tp["quat"][tr]
            dp["log_scale"][dr] = clone_ls
            dp["opacity_logit"][dr] = new_logit
            dp["color"][dr] = tp["color"][tr]
            for k in PARAM_GROUPS:
                m_list[dg][k][dr] = 0.0
                v_list[dg][k][dr] = 0.0
        for k in PARAM_GROUPS:
            m_list[tg][k][tr] = 0.0
            v_list[tg][k][tr] = 0.0
    return len(dead)


# --------------------------------------------------------------------------
# exact ellipse-vs-tile culling (build refinement of a-4; no pixel changes)
# --------------------------------------------------------------------------

CULL_MARGIN = np.float32(64.0625)
_F = np.float32


def cull_margin(alpha, floor_log2=ALPHA_FLOOR_LOG2):
    """Per-splat maha margin M of the tile test (ss_common.cuh cull_margin):
    64.0625 (the maha <= 64 cut with a 1e-3 margin), or with the floor
    min(64.0625, (2 (f - 1) + 2 ln2 (e - floor)) (1 + 2^-10) + 2^-4) with
    alpha = f 2^e (frexp) -- an upper bound of 2 ln(alpha / 2^floor)
    (ln f <= f - 1) made of IEEE-rounded fp64 operations only, so numpy and
    the GPU agree bit for bit.  M <= 0: the splat reaches no tile."""
    alpha = np.asarray(alpha, dtype=np.float64)
    full = np.full(alpha.shape, float(CULL_MARGIN))
    if floor_log2 is None:
        return full
    f, e = np.frexp(alpha)
    m = 2.0 * (f - 1.0) + TWO_LN2 * (e - int(floor_log2)).astype(np.float64)
    m = m * 1.0009765625 + 0.0625
    m = np.minimum(m, full)
    return np.where(alpha > 0.0, m, -1.0)


def tile_geom(i0, i1, i2, margin=None):
    """Per-splat constants of the row-interval tile test, fp64 then rounded
    once to float32 (ss_common.cuh make_geom): det = i0 i2 - i1^2,
    sy = i1 sqrt(M / (i2 det)) (dy of the ellipse's rightmost point is -sy),
    ymax = sqrt(M i0 / det) (its vertical half extent), m0 = i0 M, M = the
    per-splat cull_margin (CULL_MARGIN without the alpha floor)."""
    i0, i1, i2 = (np.asarray(a, dtype=np.float64) for a in (i0, i1, i2))
    m = np.full(i0.shape, float(CULL_MARGIN)) if margin is None else np.asarray(margin, np.float64)
    mp = np.maximum(m, 0.0)  # M <= 0 reaches no tile (masked by the caller)
    det = i0 * i2 - i1 * i1
    sy = i1 * np.sqrt(mp / (i2 * det))
    ymax = np.sqrt((mp * i0) / det)
    m0 = (i0 * mp).astype(_F)
    f0 = i0.astype(_F)
    return m0, i1.astype(_F), det.astype(_F), sy.astype(_F), ymax.astype(_F), _F(1) / f0


def tile_row_span(m0, i1, det, sy, ymax, r0, v, Y0, Y1):
    """x-interval [L, R] (relative to the splat centre) where the ellipse
    m <= CULL_MARGIN meets the pixel-centre rows [Y0, Y1], and whether it
    meets them at all.  float32 restatement of ss_common.cuh row_span (same
    rounded operation sequence; numpy float32 = IEEE single without FMA).
    Tiles outside the interval hold no pixel the reference's loop blends
    (maha > 64 skip, _kernels.py:39-41)."""
    v = np.asarray(v, dtype=np.float64).astype(_F)
    lo = np.maximum(np.asarray(Y0).astype(_F) - v, -ymax)
    hi = np.minimum(np.asarray(Y1).astype(_F) - v, ymax)
    meets = lo <= hi
    cR = np.minimum(np.maximum(-sy, lo), hi)
    cL = np.minimum(np.maximum(sy, lo), hi)
    sR = np.sqrt(np.maximum(m0 - (det * cR) * cR, _F(0)))
    sL = np.sqrt(np.maximum(m0 - (det * cL) * cL, _F(0)))
    R = ((-i1) * cR + sR) * r0
    L = ((-i1) * cL - sL) * r0
    return meets, L, R


def tile_keep_mask(cache, owner, tx, ty, tile=TILE, floor_log2=ALPHA_FLOOR_LOG2):
    x0, x1, y0, y1 = cache["bbox"]
    i0, i1, i2 = cache["inv2d"][owner].T
    u, v = cache["mean2d"][owner].T
    margin = cull_margin(cache["alpha"][owner], floor_log2)
    m0, f1, det, sy, ymax, r0 = tile_geom(i0, i1, i2, margin)
    Y0 = np.maximum(ty * tile, y0[owner])
    Y1 = np.minimum(ty * tile + tile - 1, y1[owner] - 1)
    with np.errstate(invalid="ignore"):
        meets, L, R = tile_row_span(m0, f1, det, sy, ymax, r0, v, Y0, Y1)
    uf = np.asarray(u, dtype=np.float64).astype(_F)
    ax = np.maximum(tx * tile, x0[owner]).astype(_F) - uf
    bx = np.minimum(tx * tile + tile - 1, x1[owner] - 1).astype(_F) - uf
    return meets & (ax <= R) & (bx >= L) & (margin > 0.0)


# ---------------------------------------------------------------------------
# §8(f)-4 ABR tail-drop selection (server.py:39-79)

ABR_OPACITY = {0: ("<f4", 40, 56), 1: ("u1", 16, 30)}  # profile -> (dtype, byte offset, record size)
SLICE_HEADER = 16                                      # codec.py HEADER_SIZE


def abr_keep_indices(opacities, fraction):
    """server.py:39-50: ascending indices of the ceil(fraction n) highest
    opacities, ties to the lower index (stable argsort of -opacity)."""
    if not (0.0 < fraction <= 1.0):
        raise ValueError(f"fraction {fraction} outside (0, 1]")
    n = len(opacities)
    kept_n = int(math.ceil(fraction * n))
    if kept_n >= n:
        return np.arange(n)
    ranked = np.argsort(-np.asarray(opacities, dtype=np.float64), kind="stable")
    return np.sort(ranked[:kept_n])


def subsample_records(payload, profile_id, fraction):
    """server.py:59-79 on the record bytes of one slice: (kept record bytes,
    kept count).  Opacity is read at the profile's field offset (f32, or u8
    / 255 for profile 1, as the reference's astype(float64) / 255)."""
    dt, off, size = ABR_OPACITY[profile_id]
    payload = np.frombuffer(bytes(payload), dtype=np.uint8)
    n = len(payload) // size
    rec = payload.reshape(n, size)
    opac = np.frombuffer(rec[:, off:off + np.dtype(dt).itemsize].tobytes(), dtype=dt).astype(np.float64)
    if profile_id == 1:
        opac = opac / 255.0
    if fraction >= 1.0:
        return payload.tobytes(), n
    keep = abr_keep_indices(opac, fraction)
    return rec[keep].tobytes(), len(keep)
