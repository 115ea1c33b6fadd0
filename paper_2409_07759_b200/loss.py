"""Reference-facing loss API (reference loss.py:14-118) over ss_loss_l1_ssim.

``loss(pred, gt, active_optimizable, ssim_weight, opacity_reg, scale_reg)``
returns ``(LossBreakdown, grad_image, reg_grads)`` exactly like the
reference; the photometric part runs on the GPU in float32, the two
regularizer terms are O(N) host arithmetic on the given arrays (in the
trainer they are fused into the optimizer kernel instead).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .core import GaussianArrays, InvalidParameterError
from .engine import LossBuffers, device
from .raster import Image

SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2

_BUF: LossBuffers | None = None


def buffers() -> LossBuffers:
    global _BUF
    if _BUF is None:
        _BUF = LossBuffers()
    return _BUF


@dataclass
class LossBreakdown:
    total: float
    l1: float
    ssim: float
    photometric: float
    opacity_term: float
    scale_term: float


def photometric_device(pred: torch.Tensor, gt_u8=None, lut=None, gt_f32=None,
                       ssim_weight: float = 0.2, stream=None):
    """(dimg (H,W,3) f32 device, sums (2,) f64 device: sum|d|, sum SSIM)."""
    H, W = int(pred.shape[0]), int(pred.shape[1])
    return buffers().run(pred, H, W, gt_u8=gt_u8, lut=lut, gt_f32=gt_f32,
                         ssim_weight=ssim_weight, stream=stream)


def ssim_with_gradient(pred: np.ndarray, gt: np.ndarray):
    """Mean SSIM and its gradient w.r.t. pred (loss.py:35-60)."""
    dev = device()
    p = torch.from_numpy(np.ascontiguousarray(pred, dtype=np.float32)).to(dev)
    g = torch.from_numpy(np.ascontiguousarray(gt, dtype=np.float32)).to(dev)
    # ssim_weight = 1 isolates -grad(SSIM) in the image gradient
    dimg, sums = photometric_device(p, gt_f32=g, ssim_weight=1.0)
    size = pred.size
    value = float(sums[1].item()) / size
    return value, -dimg.double().cpu().numpy()


def loss(pred, gt, active_optimizable: GaussianArrays, ssim_weight: float = 0.2,
         opacity_reg: float = 2e-2, scale_reg: float = 1e-2):
    """(1-w) L1 + w (1-SSIM) + opacity_reg mean(alpha) + scale_reg mean(|s|_1)
    (loss.py:73-118)."""
    p = pred.pixels if isinstance(pred, Image) else np.asarray(pred, dtype=np.float64)
    g = gt.pixels if isinstance(gt, Image) else np.asarray(gt, dtype=np.float64)
    if p.shape != g.shape:
        raise InvalidParameterError(f"image dimensions differ: {p.shape} vs {g.shape}")
    dev = device()
    pt = torch.from_numpy(np.ascontiguousarray(p, dtype=np.float32)).to(dev)
    gtt = torch.from_numpy(np.ascontiguousarray(g, dtype=np.float32)).to(dev)
    dimg, sums = photometric_device(pt, gt_f32=gtt, ssim_weight=ssim_weight)
    s = sums.cpu().numpy()
    size = p.size
    l1 = float(s[0]) / size
    ssim_val = float(s[1]) / size
    photometric = (1.0 - ssim_weight) * l1 + ssim_weight * (1.0 - ssim_val)
    grad_image = dimg.double().cpu().numpy()
    n = len(active_optimizable)
    reg = {"opacity_logit": np.zeros((n,)), "log_scale": np.zeros((n, 3))}
    opacity_term = scale_term = 0.0
    if n > 0:
        # loss.py:105-111 on the GPU (ss_reg_grads)
        from . import _lib as L

        alpha = torch.from_numpy(np.ascontiguousarray(active_optimizable.opacities,
                                                      dtype=np.float64)).to(dev)
        scales = torch.from_numpy(np.ascontiguousarray(active_optimizable.scales,
                                                       dtype=np.float64)).to(dev)
        rl = torch.empty(n, dtype=torch.float64, device=dev)
        rs = torch.empty((n, 3), dtype=torch.float64, device=dev)
        terms = torch.empty(2, dtype=torch.float64, device=dev)
        L.check(L.lib().ss_reg_grads(L.ptr(alpha), L.ptr(scales), n, float(opacity_reg),
                                     float(scale_reg), L.ptr(rl), L.ptr(rs), L.ptr(terms),
                                     L.stream_ptr()), "reg_grads")
        opacity_term, scale_term = (float(x) for x in terms.cpu().numpy())
        reg["opacity_logit"] = rl.cpu().numpy()
        reg["log_scale"] = rs.cpu().numpy()
    total = photometric + opacity_term + scale_term
    return (LossBreakdown(total=total, l1=l1, ssim=ssim_val, photometric=photometric,
                          opacity_term=opacity_term, scale_term=scale_term), grad_image, reg)
