"""CUDA rasterizer parity against the oracle and the reference's golden vectors.

Tolerances:
  * structural (cull set, bbox, depth order, tile keys/ranges): bit-exact;
  * image: max abs <= 1e-4 (north star, on [0, 1] images);
  * gradients: per group max|d| <= 1e-3 * max|g_ref|;
  * frozen rows: exactly zero.
"""

import numpy as np
import pytest

from conftest import RASTER_CASES, arc_camera, load_golden, random_unit_quats, synth_like
from oracle import splat_oracle as O

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_REL = 1e-3


@pytest.fixture(scope="module")
def ss():
    import paper_2409_07759_b200 as P
    from paper_2409_07759_b200 import raster
    return P, raster


def cam_of(P, d):
    w, h = d["cam_wh"]
    fx, fy, cx, cy = d["cam_f"]
    return P.Camera(int(w), int(h), fx, fy, cx, cy, d["cam_R"], d["cam_T"])


def cam_from(P, c):
    return P.Camera(c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.rotation, c.translation)


def arrays_of(P, d):
    return P.GaussianArrays(d["means"], d["quats"], d["scales"], d["opacities"], d["colors"])


def grad_check(got, ref, tol=GRAD_REL, what=""):
    for k in ("mean", "log_scale", "quat", "opacity_logit", "color"):
        scale = np.abs(ref[k]).max()
        err = np.abs(got[k] - ref[k]).max()
        assert err <= tol * max(scale, 1e-30), f"{what} {k}: max|d|={err:.3e} max|ref|={scale:.3e}"


@pytest.mark.parametrize("case", RASTER_CASES)
def test_forward_matches_golden(ss, case):
    P, R = ss
    d = load_golden(f"raster_{case}")
    img = R.render_arrays(cam_of(P, d), arrays_of(P, d)).pixels
    err = np.abs(img - d["image"]).max()
    assert err <= IMG_TOL, err


@pytest.mark.parametrize("case", RASTER_CASES)
def test_backward_matches_golden(ss, case):
    P, R = ss
    d = load_golden(f"raster_{case}")
    tr = d["trainable"]
    g = R.render_arrays_backward(cam_of(P, d), arrays_of(P, d), d["grad_image"], trainable=tr)
    grad_check(g, {k: d[f"grad_{k}"] for k in g}, what=case)
    for k, v in g.items():
        assert np.all(v[~tr] == 0.0)


@pytest.mark.parametrize("case", RASTER_CASES)
def test_structural_bit_exact(ss, case):
    """Cull set, bbox and global (z, src) order equal the reference's."""
    P, R = ss
    d = load_golden(f"raster_{case}")
    R.render_arrays(cam_of(P, d), arrays_of(P, d))
    st = R.pipeline().state()
    kept = np.nonzero(st["depth_key"].numpy() != -1)[0]
    assert np.array_equal(kept, d["src"])
    assert np.array_equal(st["bbox"].numpy()[kept], d["bbox"])
    order = st["order"].numpy()[: len(kept)]
    assert np.array_equal(order, d["src"][d["order"]])


def _tile_check(P, R, cam, arrays, ocam):
    """GPU tile pairs/ranges == oracle restatement of a-4 (bit-exact, with the
    library's alpha floor).  Returns the EXACT reference bins (maha <= 64
    rule alone) for the pixel oracles: images and gradients are checked
    against the reference's own per-pixel walk."""
    R.render_arrays(cam, arrays)
    st = R.pipeline().state()
    cache = O.project_arrays(ocam, arrays.means, arrays.quats, arrays.scales, arrays.opacities,
                             arrays.colors)
    bins = O.tile_bins(cache, cam.width, cam.height, floor_log2=R.get_alpha_floor())
    assert st["n_pairs"] == bins["K"]
    keys = st["keys"].numpy().astype(np.int64)
    vals = st["vals"].numpy().astype(np.int64)
    tile_ref = (bins["keys"] >> np.uint64(O.RANK_BITS)).astype(np.int64)
    assert np.array_equal(keys, tile_ref)
    assert np.array_equal(vals, cache["src"][bins["vals"]])
    rg = st["ranges"].numpy().reshape(-1, 2)
    ref_rg = bins["ranges"].copy()
    ref_rg[ref_rg[:, 0] == ref_rg[:, 1]] = 0
    got = rg.copy()
    got[got[:, 0] == got[:, 1]] = 0
    assert np.array_equal(got, ref_rg)
    return cache, O.tile_bins(cache, cam.width, cam.height, floor_log2=None), st


@pytest.mark.parametrize("case", ["arc400", "rot1k", "saturate"])
def test_tile_keys_bit_exact_golden(ss, case):
    P, R = ss
    d = load_golden(f"raster_{case}")
    from conftest import golden_cam
    _tile_check(P, R, cam_of(P, d), arrays_of(P, d), golden_cam(d))


def _synth_scene(P, n, k, seed=0):
    rng = np.random.default_rng(seed)
    return P.GaussianArrays(*synth_like(rng, n, k))


def test_synth_medium_forward_backward_vs_oracle(ss):
    """20k synthetic splats (SURVEY §8d recipe) at 256x192 on an arc camera."""
    P, R = ss
    n = 20_000
    arr = _synth_scene(P, n, (300.0 / 30_000) ** (1 / 3), seed=1)
    ocam = arc_camera(3, 5, 256, 192)
    cam = cam_from(P, ocam)
    cache, bins, st = _tile_check(P, R, cam, arr, ocam)
    ref = O.blend_forward_tiled(cache, cam.height, cam.width, nthreads=8, bins=bins)
    img = R.render_arrays(cam, arr).pixels
    assert np.abs(img - ref["image"]).max() <= IMG_TOL
    # per-pixel contributor counts: GPU n_contrib is the list position after the
    # last contributor; the oracle reports entries walked (= same unless a break)
    gdir = np.random.default_rng(5).normal(size=(cam.height, cam.width, 3))
    g = R.render_arrays_backward(cam, arr, gdir)
    gref = O.render_arrays_backward(ocam, arr.means, arr.quats, arr.scales, arr.opacities,
                                    arr.colors, gdir, tiled=True, nthreads=8)
    grad_check(g, gref, what="synth20k")


def test_config3_crop_vs_oracle(ss):
    """300k-splat DyNeRF-shaped scene (config 3 recipe), 128x128 crop camera of
    the 1352x1014 view (shifted principal point)."""
    P, R = ss
    n = 300_000
    arr = _synth_scene(P, n, (300.0 / n) ** (1 / 3), seed=7)
    full = arc_camera(4, 20, 1352, 1014)
    from conftest import Cam
    ocam = Cam(128, 128, full.fx, full.fy, full.cx - 612, full.cy - 443, full.rotation,
               full.translation)
    cam = cam_from(P, ocam)
    cache, bins, st = _tile_check(P, R, cam, arr, ocam)
    ref = O.blend_forward_tiled(cache, cam.height, cam.width, nthreads=8, bins=bins)
    img = R.render_arrays(cam, arr).pixels
    assert np.abs(img - ref["image"]).max() <= IMG_TOL
    gdir = np.random.default_rng(6).normal(size=(cam.height, cam.width, 3)) * 1e-6
    g = R.render_arrays_backward(cam, arr, gdir)
    gref = O.projection_backward(ocam, cache, n, *O.blend_backward_tiled(
        cache, bins, cam.height, cam.width, gdir, nthreads=8))
    grad_check(g, gref, what="config3 crop")


def test_config3_full_view_structural(ss):
    """Full 1352x1014 view at 300k splats: cull set, bbox, depth order and
    every tile key bit-exact against the oracle."""
    P, R = ss
    n = 300_000
    arr = _synth_scene(P, n, (300.0 / n) ** (1 / 3), seed=7)
    ocam = arc_camera(11, 20, 1352, 1014)
    cam = cam_from(P, ocam)
    cache, bins, st = _tile_check(P, R, cam, arr, ocam)
    kept = np.nonzero(st["depth_key"].numpy() != -1)[0]
    assert np.array_equal(kept, cache["src"])
    assert np.array_equal(st["order"].numpy()[: len(kept)], cache["src"][cache["order"]])
    x0, x1, y0, y1 = cache["bbox"]
    assert np.array_equal(st["bbox"].numpy()[kept], np.stack([x0, x1, y0, y1], 1))


def test_render_deterministic(ss):
    P, R = ss
    arr = _synth_scene(P, 5000, 0.3, seed=3)
    cam = cam_from(P, arc_camera(0, 3, 200, 150))
    a = R.render_arrays(cam, arr).pixels
    b = R.render_arrays(cam, arr).pixels
    assert np.array_equal(a, b)


def test_empty_and_all_culled(ss):
    P, R = ss
    cam = P.Camera(32, 32, 60.0, 60.0, 16.0, 16.0, np.eye(3), np.zeros(3))
    assert np.all(R.render_arrays(cam, P.GaussianArrays.empty()).pixels == 0.0)
    behind = P.GaussianArrays(np.array([[0, 0, -1.0], [5.0, 0, 2.0]]), np.tile([1.0, 0, 0, 0], (2, 1)),
                              np.full((2, 3), 0.01), np.array([0.5, 0.5]), np.full((2, 3), 0.5))
    assert np.all(R.render_arrays(cam, behind).pixels == 0.0)
    g = R.render_arrays_backward(cam, behind, np.ones((32, 32, 3)))
    assert all(np.all(v == 0) for v in g.values())


def test_single_splat_known_answers(ss):
    """test_raster.py:162-179 analytic answers, at fp32 tolerance."""
    P, R = ss
    cam = P.Camera(33, 33, 60.0, 60.0, 16.0, 16.0, np.eye(3), np.zeros(3))
    g = P.Gaussian([0, 0, 2.0], [1, 0, 0, 0], [0.05] * 3, 0.37, [0.8, 0.5, 0.1])
    img = R.render(cam, [(g, P.Lifespan(0, 0, 10))], frame=0).pixels
    np.testing.assert_allclose(img[16, 16], np.array([0.8, 0.5, 0.1]) * 0.37, rtol=1e-6)
    a, b = 0.4, 0.3
    g1 = P.Gaussian([0, 0, 2.0], [1, 0, 0, 0], [0.05] * 3, a, [1.0, 0.0, 0.0])
    g2 = P.Gaussian([0, 0, 2.5], [1, 0, 0, 0], [0.05] * 3, b, [0.0, 1.0, 0.0])
    ls = P.Lifespan(0, 0, 10)
    img = R.render(cam, [(g1, ls), (g2, ls)], frame=0).pixels
    np.testing.assert_allclose(img[16, 16, 0], a, rtol=1e-6)
    np.testing.assert_allclose(img[16, 16, 1], b * (1 - a), rtol=1e-6)


def test_active_filter_and_consistency_error(ss):
    P, R = ss
    rng = np.random.default_rng(12345)
    from conftest import random_unit_quats as ruq
    arr = P.GaussianArrays(rng.uniform((-0.5, -0.5, 2), (0.5, 0.5, 4), (12, 3)), ruq(rng, 12),
                           np.exp(rng.uniform(np.log(0.02), np.log(0.1), (12, 3))),
                           rng.uniform(0.1, 0.9, 12), rng.uniform(0, 1, (12, 3)))
    cam = P.Camera(32, 32, 60.0, 60.0, 16.0, 16.0, np.eye(3), np.zeros(3))
    spans = [P.Lifespan(0, 0, 5), P.Lifespan(2, 2, 7), P.Lifespan(5, 5, 9)]
    pairs = [(g, spans[i % 3]) for i, g in enumerate(arr.to_gaussians())]
    full = R.render(cam, pairs, 3)
    pre = R.render(cam, [p for p in pairs if p[1].start <= 3 < p[1].expire], 3)
    assert np.array_equal(full.pixels, pre.pixels)
    with pytest.raises(R.ConsistencyError):
        R.render_backward(cam, pairs[:4], 0, np.zeros((32, 32, 3)), expected_active=[0, 1])


def test_huge_and_tiny_splats_tile_keys_and_image(ss):
    """Splats whose 8-sigma bbox spans > 64 tiles (the emit path past the
    64-bit keep mask), sub-pixel splats, splats straddling tile borders."""
    P, R = ss
    rng = np.random.default_rng(11)
    n = 600
    means = rng.uniform((-0.6, -0.45, 1.5), (0.6, 0.45, 3.5), size=(n, 3))
    scales = np.exp(rng.uniform(np.log(0.002), np.log(0.02), size=(n, 3)))
    scales[:12] = rng.uniform(0.15, 0.35, size=(12, 3))       # huge footprints
    scales[12:40] = rng.uniform(0.0005, 0.001, size=(28, 3))  # sub-pixel
    arr = P.GaussianArrays(means, random_unit_quats(rng, n), scales, rng.uniform(0.05, 0.95, n),
                           rng.uniform(0, 1, (n, 3)))
    from conftest import Cam
    ocam = Cam(300, 220, 260.0, 250.0, 150.0, 110.0, np.eye(3), np.zeros(3))
    cam = cam_from(P, ocam)
    cache, bins, st = _tile_check(P, R, cam, arr, ocam)
    x0, x1, y0, y1 = cache["bbox"]
    ntile = (((x1 - 1) // 16) - (x0 // 16) + 1) * (((y1 - 1) // 16) - (y0 // 16) + 1)
    assert ntile.max() > 64
    ref = O.blend_forward_tiled(cache, cam.height, cam.width, nthreads=8, bins=bins)
    img = R.render_arrays(cam, arr).pixels
    assert np.abs(img - ref["image"]).max() <= IMG_TOL
    gdir = rng.normal(size=img.shape)
    g = R.render_arrays_backward(cam, arr, gdir)
    gref = O.projection_backward(ocam, cache, n, *O.blend_backward_tiled(
        cache, bins, cam.height, cam.width, gdir, nthreads=8))
    grad_check(g, gref, what="huge/tiny")


@pytest.mark.slow
def test_config3_full_view_image_and_gradients(ss):
    """A whole 1352x1014 view of the 300k-splat config-3 scene: image within
    1e-4 of the fp64 oracle everywhere, gradients within 1e-3 of the max."""
    P, R = ss
    n = 300_000
    arr = _synth_scene(P, n, (300.0 / n) ** (1 / 3), seed=7)
    ocam = arc_camera(7, 20, 1352, 1014)
    cam = cam_from(P, ocam)
    cache, bins, st = _tile_check(P, R, cam, arr, ocam)
    ref = O.blend_forward_tiled(cache, cam.height, cam.width, nthreads=O.default_threads(),
                                bins=bins)
    img = R.render_arrays(cam, arr).pixels
    err = np.abs(img - ref["image"])
    assert err.max() <= IMG_TOL, err.max()
    gdir = np.random.default_rng(3).normal(size=img.shape) * 1e-6
    g = R.render_arrays_backward(cam, arr, gdir)
    gref = O.projection_backward(ocam, cache, n, *O.blend_backward_tiled(
        cache, bins, cam.height, cam.width, gdir, nthreads=O.default_threads()))
    grad_check(g, gref, what="config3 full view")


def test_deterministic_backward_bit_identical(ss):
    """Fixed-order gradient sums: bit-identical across runs and within the
    oracle tolerance (also the >64-tile emit-position path)."""
    P, R = ss
    rng = np.random.default_rng(4)
    arr = _synth_scene(P, 20_000, (300.0 / 30_000) ** (1 / 3), seed=2)
    big = arr.scales.copy()
    big[:5] *= 8.0
    arr = P.GaussianArrays(arr.means, arr.quats, big, arr.opacities, arr.colors)
    ocam = arc_camera(1, 5, 320, 240)
    cam = cam_from(P, ocam)
    gdir = rng.normal(size=(240, 320, 3))
    R.set_deterministic(True)
    try:
        g1 = R.render_arrays_backward(cam, arr, gdir)
        g2 = R.render_arrays_backward(cam, arr, gdir)
    finally:
        R.set_deterministic(False)
    for k in g1:
        assert np.array_equal(g1[k], g2[k]), k
    gref = O.render_arrays_backward(ocam, arr.means, arr.quats, arr.scales, arr.opacities,
                                    arr.colors, gdir, tiled=True, nthreads=8)
    grad_check(g1, gref, what="deterministic")
    ga = R.render_arrays_backward(cam, arr, gdir)
    grad_check(ga, g1, tol=1e-5, what="atomic vs deterministic")


def test_forward_only_view_still_differentiable(ss):
    """ss_view.fwd_only (playback) skips the backward's aids -- entry-use
    masks and the per-tile work order: the image is bit-identical, and a
    backward run anyway (region test, the binning's tile order) matches the
    masked one up to float-atomic order."""
    P, R = ss
    rng = np.random.default_rng(9)
    arr = _synth_scene(P, 20_000, (300.0 / 30_000) ** (1 / 3), seed=5)
    cam = cam_from(P, arc_camera(2, 5, 320, 240))
    gdir = rng.normal(size=(240, 320, 3))
    img = R.render_arrays(cam, arr).pixels
    g = R.render_arrays_backward(cam, arr, gdir)
    pipe = R.pipeline()
    pipe.forward_only = True
    try:
        img_f = R.render_arrays(cam, arr).pixels
        g_f = R.render_arrays_backward(cam, arr, gdir)
        assert pipe.view.used_ok == 0
    finally:
        pipe.forward_only = False
    assert np.array_equal(img, img_f)
    grad_check(g_f, g, tol=1e-5, what="fwd_only vs masked")


def test_side_stream_tile_order_between_views(ss):
    """The backward's tile order runs on a side stream after each forward
    (ss_view.order_ready): a forward-only render of another view in between
    must not disturb the next view's backward (deterministic sums: bit
    equal to the same backward without the interleaved view)."""
    P, R = ss
    rng = np.random.default_rng(12)
    arr = _synth_scene(P, 20_000, (300.0 / 30_000) ** (1 / 3), seed=6)
    cam_a = cam_from(P, arc_camera(0, 5, 320, 240))
    cam_b = cam_from(P, arc_camera(3, 5, 256, 192))
    gdir = rng.normal(size=(192, 256, 3))
    R.set_deterministic(True)
    try:
        g_ref = R.render_arrays_backward(cam_b, arr, gdir)
        for _ in range(3):
            R.render_arrays(cam_a, arr)
        g = R.render_arrays_backward(cam_b, arr, gdir)
    finally:
        R.set_deterministic(False)
    for k in g_ref:
        assert np.array_equal(g[k], g_ref[k]), k


@pytest.mark.parametrize("n_culled", [5000, 160_000])
def test_depth_order_exact_on_adversarial_keys(n_culled):
    """ss_depth_order (range-normalised buckets + per-bucket sort) equals the
    stable 64-bit order, i.e. np.lexsort((index, z)) (raster.py:153): depths
    sharing their high 32 bits, exact ties, culled keys, long runs, runs whose
    keys share the prefix but not the high word, and far depths that clamp to
    one prefix.  n_culled = 160k: most of the store off-view, as in a novel
    view (the culled run is placed by one global atomic per CTA)."""
    import torch
    from paper_2409_07759_b200 import _lib as L
    rng = np.random.default_rng(0)
    n = 200_000
    z = rng.uniform(2.0, 3.0, n)
    z[:50_000] = 2.5 + rng.integers(0, 1000, 50_000) * 2.0 ** -44   # same high bits
    z[50_000:60_000] = 2.75                                          # exact ties
    z[60_000:61_000] = 2.75 + np.arange(1000)[::-1] * 2.0 ** -50     # long reversed run
    z[61_000:63_000] = rng.uniform(2.0 ** 14, 2.0 ** 20, 2000)             # clamped prefix
    keys = z.view(np.uint64).copy()
    # same 24-bit prefix, high words h and h + 1 (the prefix drops their last bit)
    h = (np.array([2.9]).view(np.uint64)[0] >> np.uint64(32)) & ~np.uint64(1)
    hi = h + rng.integers(0, 2, 3000).astype(np.uint64)
    keys[63_000:66_000] = (hi << np.uint64(32)) | rng.integers(0, 2 ** 32, 3000).astype(np.uint64)
    keys[rng.choice(n, n_culled, replace=False)] = np.uint64(0xFFFFFFFFFFFFFFFF)  # culled
    perm = rng.permutation(n)
    keys = keys[perm]
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    order = torch.empty(n, dtype=torch.int32, device="cuda")
    lib = L.lib()
    ws = torch.empty(int(lib.ss_binning_workspace_bytes(n, 1, 1)), dtype=torch.uint8, device="cuda")
    L.check(lib.ss_depth_order(L.ptr(kt), n, L.ptr(order), L.ptr(ws), ws.numel(),
                               L.stream_ptr()), "depth_order")
    ref = np.lexsort((np.arange(n), keys))
    got = order.cpu().numpy()
    kept = int(np.count_nonzero(keys != np.uint64(0xFFFFFFFFFFFFFFFF)))
    # the blend order is the kept prefix; culled splats follow in any order
    assert np.array_equal(got[:kept], ref[:kept])
    assert np.array_equal(np.sort(got[kept:]), np.sort(ref[kept:]))


@pytest.mark.parametrize("scene", ["config3_full", "huge"])
def test_binning_modes_agree(ss, scene):
    """Counting-sort binning (default) and emit + radix pair sort build the same
    tile lists bit for bit, hence the same image and gradients."""
    P, R = ss
    if scene == "config3_full":
        arr = _synth_scene(P, 300_000, (300.0 / 300_000) ** (1 / 3), seed=7)
        ocam = arc_camera(11, 20, 1352, 1014)
    else:
        rng = np.random.default_rng(12)
        n = 2000
        means = rng.uniform((-0.6, -0.45, 1.2), (0.6, 0.45, 3.5), size=(n, 3))
        scales = np.exp(rng.uniform(np.log(0.002), np.log(0.03), size=(n, 3)))
        scales[:30] = rng.uniform(0.2, 0.5, size=(30, 3))
        arr = P.GaussianArrays(means, random_unit_quats(rng, n), scales,
                               rng.uniform(0.05, 0.95, n), rng.uniform(0, 1, (n, 3)))
        from conftest import Cam
        ocam = Cam(700, 300, 500.0, 480.0, 350.0, 150.0, np.eye(3), np.zeros(3))
    cam = cam_from(P, ocam)
    gdir = np.random.default_rng(3).normal(size=(cam.height, cam.width, 3)) * 1e-6
    out = {}
    try:
        for mode in ("counting", "sort"):
            R.set_binning(mode)
            R.set_deterministic(True)
            img = R.render_arrays(cam, arr).pixels
            st = R.pipeline().state()
            g = R.render_arrays_backward(cam, arr, gdir)
            out[mode] = (img, st, g)
    finally:
        R.set_binning("counting")
        R.set_deterministic(False)
    (ia, sa, ga), (ib, sb, gb) = out["counting"], out["sort"]
    assert sa["n_pairs"] == sb["n_pairs"] > 0
    for k in ("keys", "vals", "ranges"):
        a, b = sa[k].numpy(), sb[k].numpy()
        if k == "ranges":
            a, b = a.reshape(-1, 2).copy(), b.reshape(-1, 2).copy()
            a[a[:, 0] == a[:, 1]] = 0
            b[b[:, 0] == b[:, 1]] = 0
        assert np.array_equal(a, b), k
    assert np.array_equal(ia, ib)
    for k in g_keys():
        assert np.array_equal(ga[k], gb[k]), k


def g_keys():
    return ("mean", "log_scale", "quat", "opacity_logit", "color")


def test_wide_frame_chunked_binning(ss):
    """A 2048x1536 frame (12288 tiles, 2/3 of the chunked binning's shared-
    memory limit): keys stay bit-exact against the oracle."""
    P, R = ss
    from paper_2409_07759_b200 import _lib as L
    rng = np.random.default_rng(23)
    n = 4000
    means = rng.uniform((-1.2, -0.9, 2.0), (1.2, 0.9, 4.0), size=(n, 3))
    scales = np.exp(rng.uniform(np.log(0.003), np.log(0.03), size=(n, 3)))
    scales[:20] = rng.uniform(0.2, 0.4, size=(20, 3))
    arr = P.GaussianArrays(means, random_unit_quats(rng, n), scales, rng.uniform(0.1, 0.9, n),
                           rng.uniform(0, 1, (n, 3)))
    from conftest import Cam
    ocam = Cam(2048, 1536, 1200.0, 1200.0, 1024.0, 768.0, np.eye(3), np.zeros(3))
    tiles = (2048 // 16) * (1536 // 16)
    assert 11 * 1024 < tiles <= 18 * 1024
    assert L.lib().ss_bin_tiles_supported(1 << 20, tiles)
    _tile_check(P, R, cam_from(P, ocam), arr, ocam)


def test_large_frame_uses_pair_sort_fallback(ss):
    """A frame with more 16x16 tiles than the chunked binning's shared-memory
    cursors hold (> 18432) falls back to emit + pair sort automatically; keys
    stay bit-exact and the image matches the oracle."""
    P, R = ss
    from paper_2409_07759_b200 import _lib as L
    rng = np.random.default_rng(21)
    n = 3000
    means = rng.uniform((-1.2, -0.9, 2.0), (1.2, 0.9, 4.0), size=(n, 3))
    scales = np.exp(rng.uniform(np.log(0.003), np.log(0.02), size=(n, 3)))
    arr = P.GaussianArrays(means, random_unit_quats(rng, n), scales, rng.uniform(0.1, 0.9, n),
                           rng.uniform(0, 1, (n, 3)))
    from conftest import Cam
    ocam = Cam(2560, 1920, 1400.0, 1400.0, 1280.0, 960.0, np.eye(3), np.zeros(3))
    tiles = (2560 // 16) * (1920 // 16)
    assert not L.lib().ss_bin_tiles_supported(1 << 20, tiles)
    cam = cam_from(P, ocam)
    cache, bins, st = _tile_check(P, R, cam, arr, ocam)
    ref = O.blend_forward_tiled(cache, cam.height, cam.width, nthreads=8, bins=bins)
    img = R.render_arrays(cam, arr).pixels
    assert np.abs(img - ref["image"]).max() <= IMG_TOL


def test_concurrent_views_from_two_threads(ss):
    """Two host threads (a trainer and a player, say), each with its own
    pipeline and stream, render different views at the same time: each view's
    pair count K arrives through its thread's own mapped word, so images equal
    the single-threaded renders bit for bit."""
    import threading

    import torch

    from paper_2409_07759_b200.engine import Store, ViewPipeline, device

    P, R = ss
    arr = _synth_scene(P, 20_000, 0.03, seed=5)
    rows = torch.from_numpy(arr.rows()).to(device())
    store = Store(opt=None, mat=rows)
    cams = [cam_from(P, arc_camera(i, 8, 320, 240)) for i in range(4)]
    ref = [ViewPipeline().forward(store, None, len(arr), c).clone() for c in cams]
    torch.cuda.synchronize()
    out = [[None] * 4 for _ in range(2)]
    errors = []

    def worker(t):
        try:
            pipe = ViewPipeline()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(5):
                    for i, c in enumerate(cams[t::2]):
                        img = pipe.forward(store, None, len(arr), c, stream=s)
                        out[t][2 * i + t] = img.clone()
            s.synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=120)
    assert not errors, errors
    for t in range(2):
        for i in range(t, 4, 2):
            assert torch.equal(out[t][i], ref[i]), (t, i)


def test_alpha_floor_off_reproduces_reference_rule(ss):
    """ss_set_alpha_floor(0): tile lists are the maha <= 64 rule alone
    (bit-exact vs the oracle's exact bins); with the default floor the lists
    shrink and the image / gradients stay within tolerance of the same
    reference walk."""
    P, R = ss
    arr = _synth_scene(P, 20_000, (300.0 / 30_000) ** (1 / 3), seed=8)
    ocam = arc_camera(2, 5, 256, 192)
    cam = cam_from(P, ocam)
    gdir = np.random.default_rng(9).normal(size=(192, 256, 3))
    default = R.get_alpha_floor()
    assert default == O.ALPHA_FLOOR_LOG2
    out = {}
    try:
        for floor in (None, default):
            R.set_alpha_floor(floor)
            assert R.get_alpha_floor() == floor
            cache, bins, st = _tile_check(P, R, cam, arr, ocam)
            img = R.render_arrays(cam, arr).pixels
            g = R.render_arrays_backward(cam, arr, gdir)
            out[floor] = (st["n_pairs"], img, g)
    finally:
        R.set_alpha_floor(default)
    ref = O.blend_forward_tiled(cache, cam.height, cam.width, nthreads=8, bins=bins)
    gref = O.projection_backward(ocam, cache, len(arr), *O.blend_backward_tiled(
        cache, bins, cam.height, cam.width, gdir, nthreads=8))
    assert out[None][0] == bins["K"] > out[default][0]
    for floor in (None, default):
        assert np.abs(out[floor][1] - ref["image"]).max() <= IMG_TOL
        grad_check(out[floor][2], gref, what=f"floor {floor}")


def test_alpha_floor_error_bound_on_deep_translucent_stack(ss):
    """Worst case for the floor: 4000 wide, faint (alpha 0.002) splats stacked
    over the same pixels, so pixels never saturate and every one of them
    skips hundreds of sub-floor fringe contributions; the image still stays
    within 1e-4 of the reference's exact walk."""
    P, R = ss
    rng = np.random.default_rng(17)
    n = 4000
    means = np.stack([rng.normal(0, 0.08, n), rng.normal(0, 0.06, n), rng.uniform(2.0, 4.0, n)], 1)
    scales = np.exp(rng.uniform(np.log(0.01), np.log(0.05), size=(n, 3)))
    arr = P.GaussianArrays(means, random_unit_quats(rng, n), scales, np.full(n, 0.002),
                           rng.uniform(0.2, 1.0, (n, 3)))
    from conftest import Cam
    ocam = Cam(160, 128, 300.0, 300.0, 80.0, 64.0, np.eye(3), np.zeros(3))
    cam = cam_from(P, ocam)
    cache, bins, st = _tile_check(P, R, cam, arr, ocam)
    ref = O.blend_forward_tiled(cache, cam.height, cam.width, nthreads=8, bins=bins)
    assert ref["t_final"].min() > 1e-4      # nothing saturates
    img = R.render_arrays(cam, arr).pixels
    assert np.abs(img - ref["image"]).max() <= IMG_TOL


def test_project_one_splat_api(ss):
    """raster.project (one splat, raster.py:176-191) through ss_project_splats:
    the reference's fp64 formulas for centre, raw covariance and depth
    (test_raster.py:64-117 style: on-axis, isotropic, culled cases)."""
    P, R = ss
    cam = P.Camera(128, 96, 100.0, 110.0, 64.0, 48.0, np.eye(3), np.zeros(3))
    g = P.Gaussian([0.0, 0.0, 3.0], [1, 0, 0, 0], [0.05] * 3, 0.5, [0.2, 0.3, 0.4])
    sp = R.project(g, cam)
    np.testing.assert_allclose(sp.mean2d, [64.0, 48.0], rtol=0, atol=1e-12)
    np.testing.assert_allclose(sp.cov2d, np.diag([(100 * 0.05 / 3) ** 2, (110 * 0.05 / 3) ** 2]),
                               rtol=1e-12)
    assert sp.depth == 3.0 and sp.opacity == 0.5
    assert R.project(P.Gaussian([0.0, 0.0, -1.0], [1, 0, 0, 0], [0.05] * 3, 0.5, [0, 0, 0]),
                     cam) is None                      # behind the camera
    assert R.project(P.Gaussian([50.0, 0.0, 3.0], [1, 0, 0, 0], [0.05] * 3, 0.5, [0, 0, 0]),
                     cam) is None                      # outside the 3-sigma cull
    rng = np.random.default_rng(3)
    for _ in range(20):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        mean = rng.uniform([-0.3, -0.3, 2.0], [0.3, 0.3, 4.0])
        s = rng.uniform(0.01, 0.1, 3)
        rot = np.array([[0.96, -0.28, 0.0], [0.28, 0.96, 0.0], [0.0, 0.0, 1.0]])
        cam2 = P.Camera(128, 96, 100.0, 110.0, 64.0, 48.0, rot, np.array([0.05, -0.02, 0.1]))
        sp = R.project(P.Gaussian(mean, q, s, 0.7, [0.5] * 3), cam2)
        t = rot @ mean + cam2.translation
        from paper_2409_07759_b200.core import quat_to_rotmat
        m3 = quat_to_rotmat(q) * s[None, :]
        J = np.array([[100.0 / t[2], 0, -100.0 * t[0] / t[2] ** 2],
                      [0, 110.0 / t[2], -110.0 * t[1] / t[2] ** 2]]) @ rot
        cov = J @ (m3 @ m3.T) @ J.T
        np.testing.assert_allclose(sp.mean2d, [100 * t[0] / t[2] + 64, 110 * t[1] / t[2] + 48],
                                   rtol=1e-12)
        np.testing.assert_allclose(sp.cov2d, cov, rtol=1e-10, atol=1e-14)
        assert sp.depth == pytest.approx(t[2], rel=1e-15)


@pytest.mark.parametrize("strips", [(2, 2), (8, 8), (4, 2), (8, 4)])
def test_raster_strips_vs_oracle(ss, strips):
    """Every strip mapping (2 / 4 / 8 pixels per lane), equal and unequal
    forward / backward strips (unequal: the entry-use masks are off), gives
    the reference's image and gradients within tolerance."""
    P, R = ss
    arr = _synth_scene(P, 12_000, (300.0 / 20_000) ** (1 / 3), seed=14)
    ocam = arc_camera(3, 6, 200, 152)
    cam = cam_from(P, ocam)
    gdir = np.random.default_rng(15).normal(size=(152, 200, 3))
    try:
        R.set_strips(*strips)
        img = R.render_arrays(cam, arr).pixels
        g = R.render_arrays_backward(cam, arr, gdir)
    finally:
        R.set_strips(4, 4)
    ref = O.render_arrays(ocam, arr.means, arr.quats, arr.scales, arr.opacities, arr.colors,
                          nthreads=8, tiled=True)
    assert np.abs(img - ref).max() <= IMG_TOL
    gref = O.render_arrays_backward(ocam, arr.means, arr.quats, arr.scales, arr.opacities,
                                    arr.colors, gdir, tiled=True, nthreads=8)
    grad_check(g, gref, what=f"strips {strips}")
