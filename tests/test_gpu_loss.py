"""Fused L1+SSIM loss kernel vs the reference golden vectors and the oracle.

Tolerances: loss terms 1e-5 relative; gradient image max|d| <= 1e-4 * max|g_ref|
(float32 SSIM statistics)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import splat_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2409_07759_b200 import loss
    return loss


def test_loss_matches_golden(L):
    import paper_2409_07759_b200 as P
    d = load_golden("loss")
    n = len(d["opacities"])
    arr = P.GaussianArrays(np.zeros((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), d["scales"],
                           d["opacities"], np.zeros((n, 3)))
    br, grad, reg = L.loss(d["pred"], d["gt"], arr)
    ref = d["breakdown"]
    got = [br.total, br.l1, br.ssim, br.photometric, br.opacity_term, br.scale_term]
    np.testing.assert_allclose(got, ref, rtol=1e-5)
    scale = np.abs(d["grad_image"]).max()
    assert np.abs(grad - d["grad_image"]).max() <= 1e-4 * scale
    np.testing.assert_allclose(reg["opacity_logit"], d["reg_opacity_logit"], rtol=1e-12)
    np.testing.assert_allclose(reg["log_scale"], d["reg_log_scale"], rtol=1e-12)
    v, g = L.ssim_with_gradient(d["pred"], d["gt"])
    assert v == pytest.approx(float(d["ssim_value"]), rel=1e-5)
    assert np.abs(g - d["ssim_grad"]).max() <= 1e-4 * np.abs(d["ssim_grad"]).max()


@pytest.mark.parametrize("shape", [(200, 260), (1014, 1352), (37, 53)])
def test_loss_u8_ground_truth_vs_oracle(shape):
    """u8 sRGB ground truth through the LUT (read_png semantics) at several sizes,
    including DyNeRF resolution and non-multiple-of-32 edges."""
    import torch
    from paper_2409_07759_b200 import loss as L
    from paper_2409_07759_b200.raster import srgb_u8_lut
    H, W = shape
    rng = np.random.default_rng(H)
    pred = rng.uniform(0, 1, size=(H, W, 3))
    gt_u8 = rng.integers(0, 256, size=(H, W, 3), dtype=np.uint8)
    # the kernel sees float32 LUT values; give the oracle the same inputs so
    # sign(pred - gt) ties resolve identically
    gt = O.linear_from_u8(gt_u8).astype(np.float32).astype(np.float64)
    pred32 = pred.astype(np.float32)
    br, gref, _ = O.loss(pred32.astype(np.float64), gt, np.zeros(0), np.zeros((0, 3)))
    dev = torch.device("cuda")
    lut = torch.from_numpy(srgb_u8_lut().astype(np.float32)).to(dev)
    dimg, sums = L.photometric_device(torch.from_numpy(pred32).to(dev),
                                      gt_u8=torch.from_numpy(gt_u8).to(dev), lut=lut)
    s = sums.cpu().numpy() / pred.size
    assert s[0] == pytest.approx(br["l1"], rel=1e-5)
    assert s[1] == pytest.approx(br["ssim"], rel=1e-5)
    g = dimg.double().cpu().numpy()
    assert np.abs(g - gref).max() <= 1e-4 * np.abs(gref).max()
