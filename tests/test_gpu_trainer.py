"""Device trainer state vs the reference semantics: active-set compaction
(a-2, bit-exact index order), maturation / export through the device store
(a-13), and relocation / SGLD on the device path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    from paper_2409_07759_b200 import train
    return train


def _state(T, swin=4, num_gs=40, seed=3, **kw):
    cfg = T.TrainConfig(swin_size=swin, num_gs=num_gs, genesis_iterations=2, window_iterations=1,
                        rng_seed=seed, **kw)
    st = T.init_state(cfg)
    st.genesis_done = True
    return st


def _expected_rows(state, frame):
    """Reference order (train.py:380-386): optimizable generations in
    state.slices order, then matured generations in archive order."""
    sl = state.config.slice_size
    n_opt = state.config.num_gs
    rows = []
    for i, g in enumerate(state.slices):
        if g.lifespan.start <= frame < g.lifespan.expire:
            rows += list(range(i * sl, (i + 1) * sl))
    n_opt_act = len(rows)
    for m in state.matured:
        if m.lifespan.start <= frame < m.lifespan.expire:
            rows += list(range(n_opt + m.block * sl, n_opt + (m.block + 1) * sl))
    return rows, n_opt_act


def test_compaction_bit_exact_through_window_slides(T):
    state = _state(T)
    T.schedule_expire(state)
    model = state.to_device()
    for st in range(1, 12):
        T.mature(st, state, writer=None)
        for frame in range(max(0, st - 5), st + 6):
            rows, n, n_opt = model.compact(frame)
            exp, exp_opt = _expected_rows(state, frame)
            assert n == len(exp) and n_opt == exp_opt
            got = rows[:n].cpu().numpy().tolist()
            assert got == exp, (st, frame)
            counts = model.counts.cpu().numpy()
            assert counts[0] == len(exp) and counts[1] == exp_opt
        if st == 1:  # partition after the first rebirth (test_trainer.py:314-328)
            for frame in range(1, 5):
                assert model.compact(frame)[1] == state.config.num_gs


def test_compaction_empty_and_large(T):
    import torch
    from paper_2409_07759_b200 import _lib as L
    lib = L.lib()
    for n_opt, n_mat, bl in ((0, 0, 1), (5000, 0, 1000), (0, 3000, 1000), (123457, 20000, 4000)):
        rng = np.random.default_rng(n_opt + n_mat)
        tot = n_opt + n_mat + bl
        start = torch.from_numpy(rng.integers(0, 5, tot).astype(np.int32)).cuda()
        expire = start + torch.from_numpy(rng.integers(0, 5, tot).astype(np.int32)).cuda()
        nb = max(1, (n_mat + bl - 1) // bl) + 1
        perm = rng.permutation(nb).astype(np.int32)
        blk = torch.from_numpy(perm).cuda()
        out = torch.empty(tot + 1, dtype=torch.int32, device="cuda")
        counts = torch.zeros(2, dtype=torch.int32, device="cuda")
        ws = torch.empty(int(lib.ss_compact_workspace_bytes(n_opt + n_mat)), dtype=torch.uint8,
                         device="cuda")
        frame = 2
        L.check(lib.ss_compact_active(L.ptr(start), L.ptr(expire), n_opt, n_mat, L.ptr(blk), bl,
                                      frame, L.ptr(out), L.ptr(counts), L.ptr(ws), ws.numel(),
                                      L.stream_ptr()), "compact")
        s, e = start.cpu().numpy(), expire.cpu().numpy()
        cand = list(range(n_opt)) + [n_opt + perm[c // bl] * bl + c % bl for c in range(n_mat)]
        exp = [c for c in cand if s[c] <= frame < e[c]]
        c = counts.cpu().numpy()
        assert c[0] == len(exp) and c[1] == sum(1 for x in exp if x < n_opt)
        assert out[: len(exp)].cpu().numpy().tolist() == exp


def test_device_mature_export_matches_host_encode(T, tmp_path):
    """Frozen generations snapshot through ss_to_direct equal the reference's
    gen.arrays() (exp / sigmoid on the host) to the last ulp or two, and the
    emitted bytes re-encode identically from the archive."""
    from paper_2409_07759_b200.codec import PROFILES, pack_slice
    state = _state(T, swin=2, num_gs=20, profile_id=1)
    host = {i: {k: v.copy() for k, v in g.params.items()} for i, g in enumerate(state.slices)}
    T.schedule_expire(state)
    state.to_device()
    blobs, archive = [], []

    class W:
        def write_slice(self, b):
            blobs.append(b)

    T.mature(1, state, W(), keep_archive=archive)
    for frozen in archive:  # (birth, slot) order
        p = host[[i for i, g in enumerate(state.slices) if g.slot == frozen.slot][0]]
        np.testing.assert_allclose(frozen.arrays.scales, np.exp(p["log_scale"]), rtol=1e-15)
        np.testing.assert_allclose(frozen.arrays.opacities, 1 / (1 + np.exp(-p["opacity_logit"])),
                                   rtol=1e-15)
        np.testing.assert_array_equal(frozen.arrays.means, p["mean"])
    for frozen, blob in zip(archive, blobs):
        assert pack_slice(frozen.arrays, frozen.lifespan, PROFILES[1], 2) == blob


def test_device_sgld_noise_statistics(T):
    """Philox SGLD on the device path: noise covariance proportional to the
    splat covariance (test_trainer.py:111-136 Monte-Carlo oracle)."""
    import torch
    from paper_2409_07759_b200 import _lib as L
    from paper_2409_07759_b200.core import covariance, quat_to_rotmat
    from paper_2409_07759_b200.device_model import _hyper
    n = 20000
    q = np.array([0.8, 0.3, -0.4, 0.33])
    q /= np.linalg.norm(q)
    s = np.array([0.3, 0.1, 0.05])
    alpha = 0.002
    row = np.concatenate([np.zeros(3), q, np.log(s), [np.log(alpha / (1 - alpha))], [0.5] * 3])
    opt = torch.from_numpy(np.tile(row, (n, 1))).cuda()
    cfg = T.TrainConfig()
    h = _hyper(cfg, 1, True, 1234, 7)
    tab = np.zeros(1, dtype=[("active", "<i4"), ("pad", "<i4"), ("bc1", "<f8"), ("bc2", "<f8"),
                             ("gscale", "<f8")])
    tab["active"] = 1
    tab_t = torch.from_numpy(tab.view(np.uint8)).cuda()
    import ctypes
    L.check(L.lib().ss_sgld(L.ptr(opt), n, n, L.ptr(tab_t), ctypes.byref(h), None,
                            L.stream_ptr()), "sgld")
    d = opt[:, :3].cpu().numpy()
    gate = 1.0 / (1.0 + np.exp(100.0 * (alpha - 0.005)))
    gain = cfg.noise_lr * cfg.lr_mean * gate
    cov = d.T @ d / n / gain ** 2
    sigma = covariance(q, s)
    assert np.linalg.norm(cov - sigma) / np.linalg.norm(sigma) < 0.05
    assert abs(d.mean(axis=0)).max() < 4 * gain * s.max() / np.sqrt(n)


def test_device_relocation_conserves_and_revives(T):
    """Philox relocation inside the device model: dead splats are re-seeded onto
    alive ones with the opacity formula, counts and lifespans unchanged."""
    import torch
    state = _state(T, swin=2, num_gs=2000, seed=9)
    rng = np.random.default_rng(0)
    for g in state.slices:
        a = rng.uniform(0.001, 0.9, len(g.params["mean"]))
        a[:50] = 0.001
        g.params["opacity_logit"][:] = np.log(a / (1 - a))
    model = state.to_device()
    model._gen_table([True, True])
    before = model.opt.clone()
    model.relocate_device(0.005)
    torch.cuda.synchronize()
    after = model.opt
    alpha_b = 1 / (1 + torch.exp(-before[:, 10]))
    alpha_a = 1 / (1 + torch.exp(-after[:, 10]))
    dead = (alpha_b < 0.005).nonzero().flatten()
    assert len(dead) >= 100
    c = model.reloc_counts.cpu().numpy()
    assert c[0] == len(dead) and c[1] == 2000 - len(dead)
    # every relocated row copies an alive target's mean exactly
    alive_means = {tuple(x) for x in before[alpha_b >= 0.005, :3].cpu().numpy().tolist()}
    for r in dead.cpu().numpy()[:200]:
        assert tuple(after[r, :3].cpu().numpy().tolist()) in alive_means
    assert after.shape == before.shape


def test_deterministic_training_is_bit_reproducible(T, tmp_path):
    """With fixed-order gradient sums the whole device step (render, loss,
    backward, Adam + Philox SGLD, relocation) is bit-reproducible: two
    train_video runs write identical containers (test_trainer.py:468-473)."""
    import paper_2409_07759_b200 as P
    from paper_2409_07759_b200 import synth
    _, ds = synth.synth_scene(3, 5, 2, 300, tmp_path / "ds", width=48, height=40)
    cfg = T.TrainConfig(swin_size=2, num_gs=200, genesis_iterations=12, window_iterations=6,
                        relocate_period=5, rng_seed=0, max_cached_frames=4)
    T.train_video(ds, cfg, tmp_path / "a.swin", deterministic=True)
    ds2 = type(ds)(tmp_path / "ds", max_cached_frames=4)
    T.train_video(ds2, cfg, tmp_path / "b.swin", deterministic=True)
    assert (tmp_path / "a.swin").read_bytes() == (tmp_path / "b.swin").read_bytes()


def test_ground_truth_prefetch_pipeline(T, tmp_path):
    """§8(f)-3: PNG decode on the thread pool + pinned async H2D gives exactly
    the bytes of the synchronous path; the model is independent of cache size
    and prefetching (test_trainer.py:475-484, test_dataset_synth.py:56-84)."""
    import torch
    from paper_2409_07759_b200 import synth
    from paper_2409_07759_b200.dataset import DatasetError, FrameDataset
    _, ds = synth.synth_scene(4, 6, 2, 200, tmp_path / "ds", width=40, height=32)
    pre = FrameDataset(tmp_path / "ds", max_cached_frames=1)
    keys = [(f, v) for f in range(6) for v in range(2)]
    pre.prefetch(keys + [(99, 0)])
    for f, v in keys:
        got = pre.device_frame(f, v).cpu().numpy()
        assert np.array_equal(got, ds.load_u8(f, v))
    with pytest.raises(DatasetError):
        pre.device_frame(99, 0)
    cfg = T.TrainConfig(swin_size=2, num_gs=100, genesis_iterations=6, window_iterations=4,
                        relocate_period=5, rng_seed=1, max_cached_frames=4)
    small = FrameDataset(tmp_path / "ds", max_cached_frames=1, gpu_cache_frames=1)
    T.train_video(small, cfg, tmp_path / "a.swin", deterministic=True)
    big = FrameDataset(tmp_path / "ds", max_cached_frames=1000)
    T.train_video(big, cfg, tmp_path / "b.swin", deterministic=True)
    assert (tmp_path / "a.swin").read_bytes() == (tmp_path / "b.swin").read_bytes()


def test_failure_leaves_partial_container(T, tmp_path):
    """A DatasetError mid-training leaves a container without end marker
    (test_trainer.py:514-522)."""
    from paper_2409_07759_b200 import synth
    from paper_2409_07759_b200.codec import ContainerReader
    _, ds = synth.synth_scene(7, 6, 1, 10, tmp_path / "ds", width=16, height=16)
    cfg = T.TrainConfig(swin_size=2, num_gs=20, genesis_iterations=3, window_iterations=2,
                        relocate_period=1000, rng_seed=0, max_cached_frames=4)
    ds.total_frames = 99
    with pytest.raises(Exception):
        T.train_video(ds, cfg, tmp_path / "broken.swin")
    r = ContainerReader(tmp_path / "broken.swin")
    assert not r.complete
    r.close()


def test_train_video_schedule_and_counts(T, tmp_path):
    """Schedule simulation and count conservation on the GPU trainer
    (test_trainer.py:454-495)."""
    from paper_2409_07759_b200 import synth
    from paper_2409_07759_b200.codec import ContainerReader
    _, ds = synth.synth_scene(2, 7, 1, 10, tmp_path / "ds", width=16, height=16)
    cfg = T.TrainConfig(swin_size=3, num_gs=30, genesis_iterations=3, window_iterations=2,
                        relocate_period=1000, rng_seed=0, max_cached_frames=4)
    res = T.train_video(ds, cfg, tmp_path / "c.swin", keep_archive=True)
    exp = list(range(1, 7 - 1 + 3))
    assert [e.target_frame for e in res.emitted[3:]] == exp
    assert [e.slot for e in res.emitted[3:]] == [t % 3 for t in exp]
    assert [e.slot for e in res.emitted[:3]] == [0, 1, 2]
    for frame in range(7):
        assert sum(len(m.arrays) for m in res.archive
                   if m.lifespan.start <= frame < m.lifespan.expire) == 30
    with ContainerReader(res.container_path) as r:
        assert r.complete
        recs = sum(int(g.valid.sum()) for g in r.all_generations())
        assert recs == 30 + (7 - 1) * 10 + (3 - 1) * 10
