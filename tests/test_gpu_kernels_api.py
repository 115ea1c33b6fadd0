"""`paper_2409_07759_b200._kernels` (the reference's _kernels.blend_forward /
blend_backward signatures, _kernels.py:20-130) against the oracle's C
restatement of the same loops (oracle/blend.c, pinned to the reference's
golden vectors in test_oracle_golden.py).

Tolerances as for the rasterizer: image max abs <= 1e-4; gradients per array
max|d| <= 1e-3 * max|ref|.
"""

import numpy as np
import pytest

from conftest import RASTER_CASES, golden_cam, load_golden
from oracle import splat_oracle as O

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_REL = 1e-3


@pytest.fixture(scope="module")
def K():
    from paper_2409_07759_b200 import _kernels
    return _kernels


def _cache(case):
    d = load_golden(f"raster_{case}")
    cam = golden_cam(d)
    cache = O.project_arrays(cam, d["means"], d["quats"], d["scales"], d["opacities"], d["colors"])
    return cam, cache


def _args(cache, order=None, bbox=None):
    x0, x1, y0, y1 = cache["bbox"] if bbox is None else bbox
    return (cache["order"] if order is None else order, cache["mean2d"], cache["inv2d"],
            cache["alpha"], cache["color"], x0, x1, y0, y1)


def _oracle_fwd(cache, H, W, order=None, bbox=None):
    c = dict(cache)
    if order is not None:
        c["order"] = order
    if bbox is not None:
        c["bbox"] = bbox
    return c, O.blend_forward(c, H, W, nthreads=8)


def _check_grads(got, ref, what):
    for name, g, r in zip(("g_mean2d", "g_inv2d", "g_alpha", "g_color"), got, ref):
        scale = np.abs(r).max()
        err = np.abs(g - r).max()
        assert err <= GRAD_REL * max(scale, 1e-30), f"{what} {name}: {err:.3e} vs {scale:.3e}"


@pytest.mark.parametrize("case", RASTER_CASES)
def test_blend_forward_matches_oracle(K, case):
    cam, cache = _cache(case)
    H, W = cam.height, cam.width
    img = K.blend_forward(*_args(cache), H, W)
    ref = O.blend_forward(cache, H, W, nthreads=8)
    assert img.shape == (H, W, 3) and img.dtype == np.float64
    assert np.abs(img - ref).max() <= IMG_TOL


@pytest.mark.parametrize("case", ["arc400", "rot1k", "saturate", "ties"])
def test_blend_backward_accumulates_like_oracle(K, case):
    cam, cache = _cache(case)
    H, W = cam.height, cam.width
    p = len(cache["alpha"])
    gimg = np.random.default_rng(3).normal(size=(H, W, 3))
    ref = O.blend_backward(cache, H, W, gimg, nthreads=8)
    # += contract: start from non-zero arrays
    got = [np.full((p, 2), 1.0), np.full((p, 3), 1.0), np.full(p, 1.0), np.full((p, 3), 1.0)]
    K.blend_backward(*_args(cache), H, W, gimg, *got)
    _check_grads([g - 1.0 for g in got], ref, case)


def test_explicit_bbox_and_custom_order(K):
    """Bboxes smaller than the maha <= 64 ellipse (the bbox test of
    _kernels.py:35-36 must cut pixels the ellipse still covers) and a blend
    order that is not the depth order."""
    cam, cache = _cache("rot1k")
    H, W = cam.height, cam.width
    x0, x1, y0, y1 = (np.asarray(b).copy() for b in cache["bbox"])
    rng = np.random.default_rng(9)
    shrink = rng.random(len(x0)) < 0.5
    x1[shrink] = np.maximum(x0[shrink] + 1, (x0[shrink] + x1[shrink]) // 2)
    y0[shrink] = np.minimum(y1[shrink] - 1, (y0[shrink] + y1[shrink]) // 2)
    bbox = (x0, x1, y0, y1)
    order = rng.permutation(np.asarray(cache["order"]))[: len(cache["order"]) * 3 // 4]
    c, ref = _oracle_fwd(cache, H, W, order=order, bbox=bbox)
    img = K.blend_forward(*_args(cache, order=order, bbox=bbox), H, W)
    assert np.abs(img - ref).max() <= IMG_TOL
    gimg = rng.normal(size=(H, W, 3))
    refg = O.blend_backward(c, H, W, gimg, nthreads=8)
    p = len(cache["alpha"])
    got = [np.zeros((p, 2)), np.zeros((p, 3)), np.zeros(p), np.zeros((p, 3))]
    K.blend_backward(*_args(cache, order=order, bbox=bbox), H, W, gimg, *got)
    _check_grads(got, refg, "bbox/order")
    # splats outside `order` get no gradient
    out = np.setdiff1d(np.arange(p), order)
    assert all(np.all(g[out] == 0) for g in got)


def test_empty_order_and_errors(K):
    from paper_2409_07759_b200.core import InvalidParameterError
    cam, cache = _cache("arc400")
    H, W = cam.height, cam.width
    img = K.blend_forward(*_args(cache, order=np.zeros(0, dtype=np.int64)), H, W)
    assert np.all(img == 0)
    with pytest.raises(InvalidParameterError):
        K.blend_forward(*_args(cache, order=np.array([0, 0])), H, W)
    with pytest.raises(InvalidParameterError):
        K.blend_backward(*_args(cache), H, W, np.zeros((H + 1, W, 3)),
                         np.zeros((1, 2)), np.zeros((1, 3)), np.zeros(1), np.zeros((1, 3)))
