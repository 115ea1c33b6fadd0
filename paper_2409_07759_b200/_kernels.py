"""The reference's pixel-loop kernels (reference _kernels.py:20-130) with the
same names, arguments and contracts, on the CUDA view pipeline:

* ``blend_forward(order, mean2d, inv2d, alpha, color, x0, x1, y0, y1, height,
  width) -> (H, W, 3) float64``                                 (_kernels.py:20-53)
* ``blend_backward(order, mean2d, inv2d, alpha, color, x0, x1, y0, y1, height,
  width, grad_img, g_mean2d, g_inv2d, g_alpha, g_color) -> None`` adds into the
  caller's zeroed arrays                                        (_kernels.py:56-130)

Per pixel the splats of ``order`` are walked with the reference's rules (bbox
test, maha > 64 skip, alpha' = min(alpha G, 0.999), stop once T < 1e-4).  The
splats are binned into 16x16 tiles in ``order`` (ss_render2d_fwd: depth key =
position in ``order``), so each pixel sees exactly the reference's sequence;
blending is fp32 (image within 1e-4, gradients within 1e-3 of max, the
north-star tolerances).  ``order`` must not repeat a splat.
"""

from __future__ import annotations

import numpy as np
import torch

from .core import InvalidParameterError
from .engine import Splats2D, ViewPipeline, device

ALPHA_MAX = 0.999   # _kernels.py:14
T_MIN = 1e-4        # _kernels.py:15
MAHA_MAX = 64.0     # _kernels.py:16

_PIPE: ViewPipeline | None = None


def _pipe() -> ViewPipeline:
    global _PIPE
    if _PIPE is None:
        _PIPE = ViewPipeline()
    return _PIPE


def _splats(order, mean2d, inv2d, alpha, color, x0, x1, y0, y1) -> Splats2D:
    dev = device()
    alpha = np.ascontiguousarray(alpha, dtype=np.float64).reshape(-1)
    n = alpha.shape[0]
    mean2d = np.ascontiguousarray(mean2d, dtype=np.float64).reshape(n, 2)
    inv2d = np.ascontiguousarray(inv2d, dtype=np.float64).reshape(n, 3)
    color = np.ascontiguousarray(color, dtype=np.float64).reshape(n, 3)
    order = np.asarray(order, dtype=np.int64).reshape(-1)
    if order.size and (order.min() < 0 or order.max() >= n):
        raise InvalidParameterError("order holds an index outside the splat arrays")
    rank = np.full(n, -1, dtype=np.int32)
    rank[order] = np.arange(order.size, dtype=np.int32)
    if np.count_nonzero(rank >= 0) != order.size:
        raise InvalidParameterError("order repeats a splat")
    bbox = np.stack([np.asarray(b, dtype=np.int64).reshape(-1) for b in (x0, x1, y0, y1)], 1)
    bbox = np.clip(bbox, -(1 << 30), 1 << 30).astype(np.int32)

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    return Splats2D(up(mean2d), up(inv2d), up(alpha), up(color), up(bbox), up(rank))


def blend_forward(order, mean2d, inv2d, alpha, color, x0, x1, y0, y1, height, width):
    """Front-to-back alpha blending; returns an (H, W, 3) float64 image."""
    height, width = int(height), int(width)
    if height <= 0 or width <= 0:
        return np.zeros((max(height, 0), max(width, 0), 3))
    sp = _splats(order, mean2d, inv2d, alpha, color, x0, x1, y0, y1)
    img = _pipe().forward2d(sp, width, height)
    return img.double().cpu().numpy()


def blend_backward(order, mean2d, inv2d, alpha, color, x0, x1, y0, y1, height, width, grad_img,
                   g_mean2d, g_inv2d, g_alpha, g_color):
    """Add dLoss/d(mean2d, inv2d, alpha, color) for dLoss/dpixels = grad_img
    into the four caller-owned arrays (reference: in-place +=)."""
    height, width = int(height), int(width)
    grad_img = np.ascontiguousarray(grad_img, dtype=np.float64)
    if grad_img.shape != (height, width, 3):
        raise InvalidParameterError(f"grad_img shape {grad_img.shape} != ({height}, {width}, 3)")
    sp = _splats(order, mean2d, inv2d, alpha, color, x0, x1, y0, y1)
    if sp.n == 0 or height == 0 or width == 0:
        return
    pipe = _pipe()
    pipe.forward2d(sp, width, height)
    dev = device()
    n = sp.n
    outs = [torch.zeros(shape, dtype=torch.float64, device=dev)
            for shape in ((n, 2), (n, 3), (n,), (n, 3))]
    dimg = torch.from_numpy(grad_img.astype(np.float32)).to(dev)
    pipe.backward2d(dimg, *outs)
    for host, d in zip((g_mean2d, g_inv2d, g_alpha, g_color), outs):
        host += d.cpu().numpy().reshape(host.shape)
