"""Fused optimizer / SGLD / relocation kernels and the GPU trainer vs the
reference's golden vectors (tests/golden/optim.npz, train_tiny.npz).

Tolerances: SGLD and relocation with injected draws <= 1e-12 relative
(fp64 kernels; libm ulp differences only); Adam with float32 gradients
(the trainer's gradient buffer) <= 1e-6 relative on moments and 1e-8
absolute on parameters."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
GROUPS = ("mean", "quat", "log_scale", "opacity_logit", "color")


@pytest.fixture(scope="module")
def T():
    from paper_2409_07759_b200 import train
    return train


def _gen(T, d, prefix, gi):
    import paper_2409_07759_b200 as P
    params = {k: d[f"{prefix}_{gi}_{k}"].copy() for k in GROUPS}
    return T.SliceGen(slot=gi, lifespan=P.Lifespan(0, 0, 5), params=params)


def test_adam_steps_match_reference(T):
    d = load_golden("optim")
    ng = int(d["n_gens"])
    gens = [_gen(T, d, "p0", gi) for gi in range(ng)]
    gens[2].adam_t = 7
    cfg = T.TrainConfig(swin_size=5, num_gs=500)
    for step in range(2):
        for gi, g in enumerate(gens):
            grads = {k: d[f"g{step}_{gi}_{k}"] for k in GROUPS}
            T._optimizer_step(g, grads, cfg)
            assert g.adam_t == int(d[f"t{step}_{gi}"])
            for k in GROUPS:
                np.testing.assert_allclose(g.params[k], d[f"p{step + 1}_{gi}_{k}"], rtol=0, atol=1e-8)
                for mom, key in ((g.adam_m, "m"), (g.adam_v, "v")):
                    ref = d[f"{key}{step + 1}_{gi}_{k}"]
                    np.testing.assert_allclose(mom[k], ref, rtol=1e-6,
                                               atol=1e-6 * np.abs(ref).max())


def test_sgd_step_matches_reference(T):
    d = load_golden("optim")
    g = _gen(T, d, "p2", 0)
    T._optimizer_step(g, {k: d[f"g1_0_{k}"] for k in GROUPS},
                      T.TrainConfig(swin_size=5, num_gs=500, optimizer="sgd"))
    for k in GROUPS:
        np.testing.assert_allclose(g.params[k], d[f"sgd_{k}"], rtol=0, atol=1e-8)


def test_sgld_matches_reference_with_same_draws(T):
    d = load_golden("optim")
    ng = int(d["n_gens"])
    gens = [_gen(T, d, "p2", gi) for gi in range(ng)]
    T.sgld_perturb(gens, 1.6e-4, 5e4, np.random.default_rng(99))
    for gi in range(ng):
        np.testing.assert_allclose(gens[gi].params["mean"], d[f"sgld_mean_{gi}"], rtol=1e-12,
                                   atol=1e-15)


def test_relocation_matches_reference_with_same_uniforms(T):
    d = load_golden("optim")
    ng = int(d["n_gens"])
    gens = []
    for gi in range(ng):
        g = _gen(T, d, "pre_reloc", gi)
        for k in GROUPS:
            g.adam_m[k][...] = d[f"pre_reloc_m_{gi}_{k}"]
            g.adam_v[k][...] = d[f"pre_reloc_v_{gi}_{k}"]
        gens.append(g)
    moved = T.relocate(gens, 0.3, np.random.default_rng(5))
    assert moved == int(d["reloc_moved"])
    for gi in range(ng):
        for k in GROUPS:
            np.testing.assert_allclose(gens[gi].params[k], d[f"post_reloc_{gi}_{k}"], rtol=1e-12,
                                       atol=1e-14, err_msg=f"{gi} {k}")
            assert np.array_equal(gens[gi].adam_m[k] == 0, d[f"post_reloc_m_{gi}_{k}"] == 0)


def test_relocation_count_and_membership_conserved(T):
    import paper_2409_07759_b200 as P
    rng = np.random.default_rng(2)
    gens = []
    for i in range(3):
        n = 15
        q = rng.normal(size=(n, 4))
        params = {"mean": rng.uniform(-1, 1, (n, 3)), "quat": q / np.linalg.norm(q, axis=1, keepdims=True),
                  "log_scale": np.log(rng.uniform(0.02, 0.1, (n, 3))),
                  "opacity_logit": T._logit(rng.uniform(0.001, 0.9, n)), "color": rng.uniform(0, 1, (n, 3))}
        gens.append(T.SliceGen(slot=i, lifespan=P.Lifespan(i, i, i + 5), params=params))
    spans = [g.lifespan for g in gens]
    T.relocate(gens, 0.05, np.random.default_rng(2))
    assert [len(g.params["mean"]) for g in gens] == [15] * 3
    assert [g.lifespan for g in gens] == spans


def test_train_swin_matches_reference_tiny(T):
    """Three genesis iterations of the reference trainer (train_tiny.npz) vs the
    GPU trainer in the reference's numpy draw order.  Float32 rendering makes
    gradients differ at ~1e-6 relative; Adam's first steps are sign-like, so
    parameters agree except where a gradient is within fp32 noise of zero."""
    import paper_2409_07759_b200 as P
    from paper_2409_07759_b200.dataset import DeviceVideoDataset
    from paper_2409_07759_b200.raster import to_u8
    import torch
    d = load_golden("train_tiny")
    n_views = int(d["cam_count"])
    cams = []
    for v in range(n_views):
        w, h = d[f"cam{v}_wh"]
        fx, fy, cx, cy = d[f"cam{v}_f"]
        cams.append(P.Camera(int(w), int(h), fx, fy, cx, cy, d[f"cam{v}_R"], d[f"cam{v}_T"]))
    gts = d["gt"]
    ds = DeviceVideoDataset(cams, gts.shape[0],
                            lambda f, v: torch.from_numpy(to_u8(gts[f, v])).cuda())
    cfg = T.TrainConfig(swin_size=2, num_gs=40, genesis_iterations=3, window_iterations=2,
                        relocate_period=2, rng_seed=11)
    state = T.init_state(cfg)
    state.noise_source = "numpy"
    for gi, g in enumerate(state.slices):
        for k in GROUPS:
            np.testing.assert_array_equal(g.params[k], d[f"init_{gi}_{k}"])
    T.train_swin(0, cfg.swin_size, state, ds)
    total = bad = 0
    for gi, g in enumerate(state.slices):
        assert g.adam_t == int(d[f"final_t_{gi}"])
        for k in GROUPS:
            got = g.params[k].cpu().numpy()
            ref = d[f"final_{gi}_{k}"]
            lr = cfg.group_lr(k)
            diff = np.abs(got - ref)
            assert diff.max() <= 6 * lr + 1e-12, (gi, k, diff.max())
            total += diff.size
            bad += int((diff > 1e-6 * max(1.0, np.abs(ref).max())).sum())
    assert bad <= 0.02 * total, (bad, total)


def test_train_window_slides_match_reference(T):
    """Past genesis (train_window.npz, the reference trainer itself): two
    window slides with maturation -- views mix optimizable and matured rows
    -- relocation at it = 0 and 2 of each window, and a surviving generation
    trained with gamma^w = 0.5 (train.py:353-506).  GPU trainer in the
    reference's numpy draw order; tolerance as the genesis test (fp32
    gradients, sign-like early Adam steps)."""
    import paper_2409_07759_b200 as P
    from paper_2409_07759_b200.dataset import DeviceVideoDataset
    from paper_2409_07759_b200.raster import to_u8
    import torch
    d = load_golden("train_window")
    cams = []
    for v in range(int(d["cam_count"])):
        w, h = d[f"cam{v}_wh"]
        fx, fy, cx, cy = d[f"cam{v}_f"]
        cams.append(P.Camera(int(w), int(h), fx, fy, cx, cy, d[f"cam{v}_R"], d[f"cam{v}_T"]))
    gts = d["gt"]
    ds = DeviceVideoDataset(cams, gts.shape[0],
                            lambda f, v: torch.from_numpy(to_u8(gts[f, v])).cuda())
    cfg = T.TrainConfig(swin_size=2, num_gs=60, genesis_iterations=3, window_iterations=4,
                        relocate_period=2, rng_seed=13)
    state = T.init_state(cfg)
    state.noise_source = "numpy"

    def check(tag):
        total = bad = 0
        for gi, g in enumerate(state.slices):
            assert g.adam_t == int(d[f"{tag}_t_{gi}"]), (tag, gi)
            assert g.windows_trained == int(d[f"{tag}_w_{gi}"]), (tag, gi)
            assert [g.lifespan.birth, g.lifespan.start, g.lifespan.expire] == \
                d[f"{tag}_life_{gi}"].tolist()
            for k in GROUPS:
                got = g.params[k].cpu().numpy()
                ref = d[f"{tag}_{gi}_{k}"]
                diff = np.abs(got - ref)
                assert diff.max() <= 12 * cfg.group_lr(k) + 1e-12, (tag, gi, k, diff.max())
                total += diff.size
                bad += int((diff > 1e-6 * max(1.0, np.abs(ref).max())).sum())
        assert len(state.matured) == int(d[f"{tag}_n_matured"])
        for mi, m in enumerate(state.matured):
            a = m.arrays
            rows = np.concatenate([a.means, a.quats, a.scales, a.opacities[:, None], a.colors], 1)
            ref = d[f"{tag}_mat_{mi}_rows"]
            assert np.abs(rows - ref).max() <= 0.05, (tag, mi)
            assert [m.lifespan.birth, m.lifespan.start, m.lifespan.expire] == \
                d[f"{tag}_mat_{mi}_life"].tolist()
        assert bad <= 0.05 * total, (tag, bad, total)

    T.train_swin(0, cfg.swin_size, state, ds)
    check("genesis")
    T.schedule_expire(state)
    T.mature(1, state, writer=None)
    T.train_swin(1, 1 + cfg.swin_size, state, ds)
    check("w1")
    T.mature(2, state, writer=None)
    T.train_swin(2, 2 + cfg.swin_size, state, ds, iterations=3)
    check("w2")


def test_relocation_large_matches_oracle_with_same_uniforms(T):
    """ss_relocate's own partition / scan kernels (no library code) at scale:
    6 generations x 40k rows, a few percent dead, the reference's uniforms;
    the post-state equals the oracle's relocate (train.py:267-318) to 1e-12,
    moments of relocated rows zeroed, counts conserved."""
    import paper_2409_07759_b200 as P
    from oracle import splat_oracle as O
    rng = np.random.default_rng(31)
    gens, ref_params, ref_m, ref_v = [], [], [], []
    for i in range(6):
        n = 40_000
        q = rng.normal(size=(n, 4))
        a = rng.uniform(0.0005, 0.95, n)
        dead = rng.random(n) < 0.03
        a[dead] = rng.uniform(1e-4, 0.004, int(dead.sum()))
        params = {"mean": rng.uniform(-1, 1, (n, 3)), "quat": q / np.linalg.norm(q, axis=1, keepdims=True),
                  "log_scale": np.log(rng.uniform(0.01, 0.1, (n, 3))),
                  "opacity_logit": T._logit(a), "color": rng.uniform(0, 1, (n, 3))}
        g = T.SliceGen(slot=i, lifespan=P.Lifespan(i, i, i + 6), params=params)
        for k in GROUPS:
            g.adam_m[k][...] = rng.normal(size=g.adam_m[k].shape)
            g.adam_v[k][...] = rng.uniform(0, 1, size=g.adam_v[k].shape)
        gens.append(g)
        ref_params.append({k: v.copy() for k, v in params.items()})
        ref_m.append({k: v.copy() for k, v in g.adam_m.items()})
        ref_v.append({k: v.copy() for k, v in g.adam_v.items()})
    alpha = np.concatenate([O.sigmoid(p["opacity_logit"]) for p in ref_params])
    n_dead = int((alpha < 0.005).sum())
    assert n_dead > 1000
    u = np.random.default_rng(7).random(n_dead)
    moved = T.relocate(gens, 0.005, np.random.default_rng(7))
    ref_moved = O.relocate(ref_params, ref_m, ref_v, 0.005, u)
    assert moved == ref_moved == n_dead
    for gi in range(6):
        for k in GROUPS:
            np.testing.assert_allclose(gens[gi].params[k], ref_params[gi][k], rtol=1e-12,
                                       atol=1e-14, err_msg=f"{gi} {k}")
            assert np.array_equal(gens[gi].adam_m[k] == 0, ref_m[gi][k] == 0)


def test_adam_tma_blocks_straddling_generations():
    """The shared-memory (TMA bulk copy) optimizer kernel: 64-row CTAs that
    straddle generations of 100 rows, half of them frozen, a tail CTA, and
    gamma^w and bias corrections that differ per generation.  Stepped rows
    match the reference step (oracle.optimizer_step: 1e-8 on parameters,
    1e-6 relative on moments); frozen rows stay bit-identical."""
    import ctypes

    import torch

    from oracle import splat_oracle as O
    from paper_2409_07759_b200 import _lib as L
    from paper_2409_07759_b200.device_model import GEN_DTYPE, _hyper, device
    from paper_2409_07759_b200.train import TrainConfig

    rng = np.random.default_rng(31)
    n_gen, sl = 10, 100
    n = n_gen * sl
    cols = {"mean": slice(0, 3), "quat": slice(3, 7), "log_scale": slice(7, 10),
            "opacity_logit": slice(10, 11), "color": slice(11, 14)}
    p = np.empty((n, 14))
    p[:, 0:3] = rng.normal(size=(n, 3))
    q = rng.normal(size=(n, 4))
    p[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    p[:, 7:10] = rng.uniform(-5, -2, size=(n, 3))
    p[:, 10] = rng.normal(size=n)
    p[:, 11:14] = rng.uniform(0, 1, size=(n, 3))
    m = rng.normal(scale=1e-3, size=(n, 14))
    v = rng.uniform(1e-8, 1e-6, size=(n, 14))
    g = rng.normal(scale=1e-2, size=(n, 14)).astype(np.float32)
    active = np.array([1, 0, 1, 1, 0, 0, 0, 1, 0, 1], dtype=np.int32)
    ts = rng.integers(0, 20, size=n_gen)
    gscale = 0.5 ** rng.integers(0, 4, size=n_gen)
    cfg = TrainConfig(swin_size=n_gen, num_gs=n)
    ocfg = dict(O.DEFAULT_CFG)
    tab = np.zeros(n_gen, dtype=GEN_DTYPE)
    for gi in range(n_gen):
        t = int(ts[gi]) + 1
        tab[gi] = (int(active[gi]), 0, 1.0 - ocfg["adam_beta1"] ** t,
                   1.0 - ocfg["adam_beta2"] ** t, float(gscale[gi]))
    dev = device()
    tp, tm, tv = (torch.from_numpy(a.copy()).to(dev) for a in (p, m, v))
    tg = torch.from_numpy(g).to(dev)
    ttab = torch.from_numpy(tab.view(np.uint8).copy()).to(dev)
    h = _hyper(cfg, 1, False, 0, 0)
    h.opacity_reg = h.scale_reg = 0.0
    L.check(L.lib().ss_adam_sgld_step(L.ptr(tp), L.ptr(tg), L.ptr(tm), L.ptr(tv), n, sl,
                                      L.ptr(ttab), ctypes.byref(h), None, L.stream_ptr()),
            "adam_sgld_step")
    gp, gm, gv = (t.cpu().numpy() for t in (tp, tm, tv))
    for gi in range(n_gen):
        r = slice(gi * sl, (gi + 1) * sl)
        if not active[gi]:
            assert np.array_equal(gp[r], p[r]) and np.array_equal(gm[r], m[r])
            assert np.array_equal(gv[r], v[r])
            continue
        grads = {k: g[r, c].astype(np.float64) for k, c in cols.items()}
        grads["mean"] = grads["mean"] * gscale[gi]
        params = {k: p[r, c].copy() for k, c in cols.items()}
        mm = {k: m[r, c].copy() for k, c in cols.items()}
        vv = {k: v[r, c].copy() for k, c in cols.items()}
        O.optimizer_step(params, mm, vv, int(ts[gi]), grads, ocfg)
        for k, c in cols.items():
            np.testing.assert_allclose(gp[r, c], params[k], rtol=0, atol=1e-8)
            np.testing.assert_allclose(gm[r, c], mm[k], rtol=1e-6, atol=1e-6 * np.abs(mm[k]).max())
            np.testing.assert_allclose(gv[r, c], vv[k], rtol=1e-6, atol=1e-6 * np.abs(vv[k]).max())
