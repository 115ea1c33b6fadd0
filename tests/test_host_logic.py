"""Host-side trainer logic that needs no GPU: config, schedule, maturation,
archive bookkeeping, and the per-iteration (frame, view) draws."""

import numpy as np
import pytest


@pytest.fixture(scope="module")
def T():
    from paper_2409_07759_b200 import train
    return train


def test_config_defaults_and_validation(T, tmp_path):
    from paper_2409_07759_b200.core import InvalidParameterError
    cfg = T.TrainConfig()
    assert (cfg.noise_lr, cfg.scale_reg, cfg.opacity_reg, cfg.ssim_weight) == (5e4, 1e-2, 2e-2, 0.2)
    assert cfg.gradient_scale_decay == 0.5 and cfg.dead_opacity_threshold == 0.005
    for bad in (dict(num_gs=10, swin_size=3), dict(window_iterations=0),
                dict(dead_opacity_threshold=1.5), dict(optimizer="lbfgs"), dict(profile_id=7)):
        with pytest.raises(InvalidParameterError):
            T.TrainConfig(**bad)
    (tmp_path / "c.json").write_text('{"swin_size": 2, "num_gs": 20}')
    assert T.TrainConfig.from_file(tmp_path / "c.json").num_gs == 20
    (tmp_path / "c.toml").write_text("swin_size = 4\nnum_gs = 40\noptimizer = 'sgd'\n")
    assert T.TrainConfig.from_file(tmp_path / "c.toml").optimizer == "sgd"
    (tmp_path / "bad.json").write_text('{"not_a_field": 1}')
    with pytest.raises(InvalidParameterError):
        T.TrainConfig.from_file(tmp_path / "bad.json")


def test_init_state_matches_reference_draws(T):
    from conftest import load_golden
    d = load_golden("train_tiny")
    cfg = T.TrainConfig(swin_size=2, num_gs=40, genesis_iterations=3, window_iterations=2,
                        relocate_period=2, rng_seed=11)
    state = T.init_state(cfg)
    for gi, g in enumerate(state.slices):
        for k in T.PARAM_GROUPS:
            np.testing.assert_array_equal(g.params[k], d[f"init_{gi}_{k}"])


def test_gradient_scale(T):
    from paper_2409_07759_b200.core import InvalidParameterError
    assert T.gradient_scale(0, 0.5) == 1.0 and T.gradient_scale(2, 0.5) == 0.25
    with pytest.raises(InvalidParameterError):
        T.gradient_scale(-1, 0.5)


def _genesis_state(T, **kw):
    cfg = T.TrainConfig(genesis_iterations=2, window_iterations=1, **kw)
    state = T.init_state(cfg)
    state.genesis_done = True  # genesis training itself needs the GPU
    return state


def test_schedule_expire(T):
    from paper_2409_07759_b200.core import StateError
    cfg = T.TrainConfig(swin_size=2, num_gs=10, genesis_iterations=1, window_iterations=1)
    with pytest.raises(StateError):
        T.schedule_expire(T.init_state(cfg))
    state = _genesis_state(T, swin_size=5, num_gs=20)
    T.schedule_expire(state)
    assert [g.lifespan.expire for g in state.slices] == [1, 2, 3, 4, 5]
    assert [g.slot for g in state.slices] == [1, 2, 3, 4, 0]
    with pytest.raises(StateError):
        T.schedule_expire(state)


def test_mature_partition_and_rebirth(T):
    state = _genesis_state(T, swin_size=5, num_gs=20)
    T.schedule_expire(state)
    emitted = []
    assert T.mature(1, state, writer=None, emitted=emitted) == 5
    for frame in range(1, 6):
        n_opt = sum(len(g.params["mean"]) for g in state.slices
                    if g.lifespan.start <= frame < g.lifespan.expire)
        n_mat = sum(len(m.arrays) for m in state.matured
                    if m.lifespan.start <= frame < m.lifespan.expire)
        assert n_opt + n_mat == 20
    for g in state.slices:
        assert g.lifespan.birth == g.lifespan.start and g.lifespan.expire - g.lifespan.start == 5
        assert g.windows_trained == 0 and g.adam_t == 0
    assert [e.slot for e in emitted] == [0, 1, 2, 3, 4]
    for st in range(2, 12):
        assert T.mature(st, state, writer=None) == 1
        assert state.matured_gaussian_count() <= 20


def test_freeze_bytes_reproducible(T):
    from paper_2409_07759_b200.codec import PROFILES, pack_slice
    state = _genesis_state(T, swin_size=2, num_gs=20, profile_id=1)
    T.schedule_expire(state)
    archive, blobs = [], []

    class W:
        def write_slice(self, b):
            blobs.append(b)

    for st in range(1, 5):
        T.mature(st, state, W(), keep_archive=archive)
    assert len(archive) == len(blobs)
    for frozen, blob in zip(archive, blobs):
        assert pack_slice(frozen.arrays, frozen.lifespan, PROFILES[1], 2) == blob


def test_sample_views_follow_reference_draw_order(T):
    cfg = T.TrainConfig(swin_size=2, num_gs=20, rng_seed=3)
    a = T.init_state(cfg)
    b = T.init_state(cfg)
    draws = T.sample_views(a, 1, 4, [0, 1, 2], 5)
    ref = [(int(b.rng.integers(1, 4)), [0, 1, 2][int(b.rng.integers(0, 3))]) for _ in range(5)]
    assert draws == ref
