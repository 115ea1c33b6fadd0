"""Pin the oracle (oracle/) against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import math

import numpy as np
import pytest

from conftest import RASTER_CASES, golden_cam, load_golden
from oracle import splat_oracle as O


def _arrays(d):
    return d["means"], d["quats"], d["scales"], d["opacities"], d["colors"]


@pytest.mark.parametrize("case", RASTER_CASES)
def test_projection_structural_bit_exact(case):
    d = load_golden(f"raster_{case}")
    cam = golden_cam(d)
    cache = O.project_arrays(cam, *_arrays(d))
    assert np.array_equal(cache["src"], d["src"])
    assert np.array_equal(cache["order"], d["order"])
    x0, x1, y0, y1 = cache["bbox"]
    assert np.array_equal(np.stack([x0, x1, y0, y1], 1), d["bbox"])
    assert np.array_equal(cache["mean2d"], d["mean2d"])
    assert np.array_equal(cache["inv2d"], d["inv2d"])


@pytest.mark.parametrize("case", RASTER_CASES)
def test_forward_matches_reference(case):
    d = load_golden(f"raster_{case}")
    cam = golden_cam(d)
    img = O.render_arrays(cam, *_arrays(d))
    np.testing.assert_allclose(img, d["image"], rtol=1e-13, atol=1e-15)
    img_t = O.render_arrays(cam, *_arrays(d), tiled=True, nthreads=4)
    np.testing.assert_allclose(img_t, d["image"], rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("case", RASTER_CASES)
def test_backward_matches_reference(case):
    d = load_golden(f"raster_{case}")
    cam = golden_cam(d)
    tr = d["trainable"]
    for tiled, nt in ((False, 1), (True, 1), (True, 3)):
        g = O.render_arrays_backward(cam, *_arrays(d), d["grad_image"], trainable=tr,
                                     tiled=tiled, nthreads=nt)
        for k in O.PARAM_GROUPS:
            ref = d[f"grad_{k}"]
            scale = max(np.abs(ref).max(), 1e-300)
            assert np.abs(g[k] - ref).max() <= 1e-11 * scale, (k, tiled, nt)
            assert np.all(g[k][~tr] == 0.0)


@pytest.mark.parametrize("floor", [None, O.ALPHA_FLOOR_LOG2])
def test_tile_bins_reproduce_reference_order(floor):
    """a-4: walking a tile's list visits the tile's splats in the reference's
    global (z, src) order restricted to that tile; a dropped splat has
    maha > 64 (or, with the alpha floor, alpha G < 2^floor) at every pixel
    of the tile."""
    d = load_golden("raster_rot1k")
    cam = golden_cam(d)
    cache = O.project_arrays(cam, *_arrays(d))
    bins = O.tile_bins(cache, cam.width, cam.height, floor_log2=floor)
    order = cache["order"]
    rank = np.empty(len(order), np.int64)
    rank[order] = np.arange(len(order))
    x0, x1, y0, y1 = cache["bbox"]
    loose = O.tile_bins(cache, cam.width, cam.height, exact=False)
    m2, inv = cache["mean2d"], cache["inv2d"]
    for t in range(bins["tiles_x"] * bins["tiles_y"]):
        s, e = bins["ranges"][t]
        lst = bins["vals"][s:e]
        assert np.all(np.diff(rank[lst]) > 0)
        tx, ty = t % bins["tiles_x"], t // bins["tiles_x"]
        hit = ((x0 < (tx + 1) * 16) & (x1 > tx * 16) & (y0 < (ty + 1) * 16) & (y1 > ty * 16)
               & (x1 > x0) & (y1 > y0))
        ls, le = loose["ranges"][t]
        assert set(np.nonzero(hit)[0]) == set(loose["vals"][ls:le].tolist())
        assert set(lst.tolist()) <= set(np.nonzero(hit)[0])
        # every dropped splat has maha > 64 at every pixel of the tile
        dropped = sorted(set(np.nonzero(hit)[0]) - set(lst.tolist()))
        ys, xs = np.mgrid[ty * 16:min(ty * 16 + 16, cam.height), tx * 16:min(tx * 16 + 16, cam.width)]
        for sidx in dropped:
            dx, dy = xs - m2[sidx, 0], ys - m2[sidx, 1]
            mm = inv[sidx, 0] * dx * dx + 2 * inv[sidx, 1] * dx * dy + inv[sidx, 2] * dy * dy
            if floor is None:
                assert mm.min() > 64.0
            else:
                ag = cache["alpha"][sidx] * np.exp(-0.5 * mm)
                assert np.all((mm > 64.0) | (ag < 2.0 ** floor))
    assert bins["K"] == len(bins["keys"]) and np.all(np.diff(bins["keys"].astype(np.float64)) >= 0)
    assert bins["K"] < loose["K"]


def test_golden_render_frontend_fixture():
    d = load_golden("golden_render")
    cam = golden_cam(d)
    parts = []
    for gi in range(int(d["n_gens"])):
        b, s, e = d[f"gen{gi}_lifespan"]
        if s <= int(d["frame"]) < e:
            v = d[f"gen{gi}_valid"]
            parts.append([d[f"gen{gi}_{k}"][v] for k in ("means", "quats", "scales", "opacities", "colors")])
    arrs = [np.concatenate([p[i] for p in parts]) for i in range(5)]
    img = O.render_arrays(cam, *arrs)
    np.testing.assert_allclose(img, d["image"], rtol=1e-13, atol=1e-15)


def test_loss_matches_reference():
    d = load_golden("loss")
    br, grad, reg = O.loss(d["pred"], d["gt"], d["opacities"], d["scales"])
    ref_br = d["breakdown"]
    got = [br[k] for k in ("total", "l1", "ssim", "photometric", "opacity_term", "scale_term")]
    np.testing.assert_allclose(got, ref_br, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(grad, d["grad_image"], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(reg["opacity_logit"], d["reg_opacity_logit"], rtol=1e-14)
    np.testing.assert_allclose(reg["log_scale"], d["reg_log_scale"], rtol=1e-14)
    v, g = O.ssim_with_gradient(d["pred"], d["gt"])
    assert v == pytest.approx(float(d["ssim_value"]), rel=1e-13)
    np.testing.assert_allclose(g, d["ssim_grad"], rtol=1e-9, atol=1e-16)


def _gen(d, prefix, gi):
    return {k: d[f"{prefix}_{gi}_{k}"].copy() for k in O.PARAM_GROUPS}


def test_optimizer_sgld_relocation_match_reference():
    d = load_golden("optim")
    ng = int(d["n_gens"])
    params = [_gen(d, "p0", gi) for gi in range(ng)]
    m = [{k: np.zeros_like(v) for k, v in p.items()} for p in params]
    v = [{k: np.zeros_like(x) for k, x in p.items()} for p in params]
    ts = [0, 0, 7]
    for step in range(2):
        for gi in range(ng):
            grads = {k: d[f"g{step}_{gi}_{k}"] for k in O.PARAM_GROUPS}
            ts[gi] = O.optimizer_step(params[gi], m[gi], v[gi], ts[gi], grads)
            assert ts[gi] == int(d[f"t{step}_{gi}"])
            for k in O.PARAM_GROUPS:
                assert np.array_equal(params[gi][k], d[f"p{step + 1}_{gi}_{k}"]), (step, gi, k)
                assert np.array_equal(m[gi][k], d[f"m{step + 1}_{gi}_{k}"])
                assert np.array_equal(v[gi][k], d[f"v{step + 1}_{gi}_{k}"])
    sgd = _gen(d, "p2", 0)
    cfg = dict(O.DEFAULT_CFG, optimizer="sgd")
    O.optimizer_step(sgd, None, None, 0, {k: d[f"g1_0_{k}"] for k in O.PARAM_GROUPS}, cfg)
    for k in O.PARAM_GROUPS:
        assert np.array_equal(sgd[k], d[f"sgd_{k}"])
    O.sgld_perturb(params, 1.6e-4, 5e4, [d[f"eta_{gi}"] for gi in range(ng)])
    for gi in range(ng):
        assert np.array_equal(params[gi]["mean"], d[f"sgld_mean_{gi}"])
    pre = [_gen(d, "pre_reloc", gi) for gi in range(ng)]
    pm = [{k: d[f"pre_reloc_m_{gi}_{k}"].copy() for k in O.PARAM_GROUPS} for gi in range(ng)]
    pv = [{k: d[f"pre_reloc_v_{gi}_{k}"].copy() for k in O.PARAM_GROUPS} for gi in range(ng)]
    moved = O.relocate(pre, pm, pv, 0.3, d["reloc_uniforms"])
    assert moved == int(d["reloc_moved"])
    for gi in range(ng):
        for k in O.PARAM_GROUPS:
            assert np.array_equal(pre[gi][k], d[f"post_reloc_{gi}_{k}"]), (gi, k)
            assert np.array_equal(pm[gi][k], d[f"post_reloc_m_{gi}_{k}"])
            assert np.array_equal(pv[gi][k], d[f"post_reloc_v_{gi}_{k}"])


def test_srgb_lut_roundtrip():
    u8 = np.arange(256, dtype=np.uint8)
    lin = O.linear_from_u8(u8)
    assert np.array_equal(O.u8_from_linear(lin), u8)
    assert lin[0] == 0.0 and lin[255] == 1.0 and np.all(np.diff(lin) > 0)


def test_abr_selection_matches_reference():
    """§8(f)-4: the oracle's abr_keep_indices / wire-level tail drop against
    the reference's own outputs (server.py:39-79, tests/golden/abr.npz)."""
    d = load_golden("abr")
    for i, q in enumerate(d["fractions"]):
        assert np.array_equal(O.abr_keep_indices(d["opac"], float(q)), d[f"keep_{i}"])
    for pid in (0, 1):
        blob = d[f"slice_p{pid}"].tobytes()
        for i, q in enumerate(d["fractions"]):
            sub = d[f"sub_p{pid}_{i}"].tobytes()
            body, kept = O.subsample_records(blob[O.SLICE_HEADER:], pid, float(q))
            assert body == sub[O.SLICE_HEADER:]
            assert len(body) == kept * O.ABR_OPACITY[pid][2]
