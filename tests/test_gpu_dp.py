"""Data-parallel training step at world_size 2, on one GPU.

Two processes (gloo over CUDA tensors: the same DataParallel.allreduce_grads
call as NCCL, SUM then x 1/G) run the real train_swin loop -- genesis window,
schedule_expire, mature, then a slid window that mixes optimizable and
matured generations, with relocation at it = 0 and every 3 iterations.  The
test asserts:
  * opt / m / v (the whole replicated device state) are bitwise equal across
    the two ranks after every phase;
  * they equal a single-process emulation of the same batch-2 semantics:
    render both ranks' draws, average the two gradient buffers ((g0 + g1) / 2,
    what the allreduce computes), then one Adam + SGLD (+ relocation) step.
Deterministic (fixed-order) gradient sums make each view's gradient
bit-reproducible, so bitwise equality is the right bar.  G = 1 reduces to
the reference loop (train.py:374-417).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SWIN, NUM_GS, FRAMES, VIEWS = 2, 600, 4, 3
GEN_IT, WIN_IT = 7, 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg(T):
    return T.TrainConfig(swin_size=SWIN, num_gs=NUM_GS, genesis_iterations=GEN_IT,
                         window_iterations=WIN_IT, relocate_period=3, rng_seed=11,
                         max_cached_frames=16)


def _snap(state):
    d = state.device
    return [t.detach().cpu().numpy().copy() for t in (d.opt, d.m, d.v)]


def _run_phases(T, state, ds, step):
    """genesis -> schedule_expire -> mature(1) -> window [1, 1 + SWIN);
    `step(st, hi, it)` runs one iteration.  Snapshots after each window."""
    out = []
    state.to_device()
    views = list(range(ds.n_views))
    for st, iters in ((0, GEN_IT), (1, WIN_IT)):
        if st == 1:
            T.schedule_expire(state)
            T.mature(1, state, writer=None)
        hi = min(st + SWIN, ds.total_frames)
        for it in range(iters):
            step(st, hi, views, it)
        for g in state.slices:
            g.windows_trained += 1
        if st == 0:
            state.genesis_done = True
        out.append(_snap(state))
    return out


def _worker(rank, world, port, root, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_07759_b200 import train as T
        from paper_2409_07759_b200.dataset import FrameDataset
        from paper_2409_07759_b200.parallel import DataParallel

        ds = FrameDataset(root, max_cached_frames=16)
        state = T.init_state(_cfg(T))
        state.deterministic = True
        state.dp = DataParallel()
        model = None

        def step(st, hi, views, it):
            nonlocal model
            model = state.device
            draws = T.sample_views(state, st, hi, views, world)
            model.train_step(draws, rank, ds, it)

        snaps = _run_phases(T, state, ds, step)
        torch.cuda.synchronize()
        out[rank] = snaps
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def dataset_root(tmp_path_factory):
    from paper_2409_07759_b200 import synth

    root = tmp_path_factory.mktemp("dp") / "ds"
    synth.synth_scene(5, FRAMES, VIEWS, 400, root, width=56, height=44)
    return root


def test_two_rank_step_replicas_equal_and_match_emulation(dataset_root):
    import torch
    import torch.multiprocessing as mp

    from paper_2409_07759_b200 import train as T
    from paper_2409_07759_b200.dataset import FrameDataset

    world = 2
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), str(dataset_root), out), nprocs=world,
                       join=True, start_method="spawn")
    r0, r1 = out[0], out[1]
    for phase in range(2):
        for a, b, name in zip(r0[phase], r1[phase], ("opt", "m", "v")):
            assert np.array_equal(a, b), f"rank replicas diverged: {name}, phase {phase}"

    # single-process emulation of the batch-2 step
    ds = FrameDataset(dataset_root, max_cached_frames=16)
    state = T.init_state(_cfg(T))
    state.deterministic = True

    def step(st, hi, views, it):
        model = state.device
        draws = T.sample_views(state, st, hi, views, world)
        stepped = T.stepped_generations(state.slices, [f for f, _ in draws])
        model._gen_table(stepped)
        acc = []
        for d in draws:
            model.view_gradients(d, ds)
            acc.append(model.grads.clone())
        model.grads.copy_(acc[0] + acc[1])
        model.grads.mul_(1.0 / world)  # DataParallel.allreduce_grads on gloo: SUM, then 1/G
        model.apply_step(stepped, it)

    emu = _run_phases(T, state, ds, step)
    torch.cuda.synchronize()
    for phase in range(2):
        for a, b, name in zip(r0[phase], emu[phase], ("opt", "m", "v")):
            assert np.array_equal(a, b), f"DP step != single-process emulation: {name}, phase {phase}"
    # the step did move the model and the matured generations exist
    assert not np.array_equal(r0[0][0], r0[1][0])
    assert len(state.matured) >= 1


def test_world1_dp_equals_plain_loop(dataset_root):
    """G = 1 through DataParallel-free train_step equals view_gradients +
    apply_step: the reference's one-view iteration (train.py:374-417)."""
    import torch

    from paper_2409_07759_b200 import train as T
    from paper_2409_07759_b200.dataset import FrameDataset

    snaps = []
    for mode in ("train_step", "parts"):
        ds = FrameDataset(dataset_root, max_cached_frames=16)
        state = T.init_state(_cfg(T))
        state.deterministic = True

        def step(st, hi, views, it, mode=mode, state=state, ds=ds):
            model = state.device
            draws = T.sample_views(state, st, hi, views, 1)
            if mode == "train_step":
                model.train_step(draws, 0, ds, it)
            else:
                stepped = T.stepped_generations(state.slices, [draws[0][0]])
                model._gen_table(stepped)
                model.view_gradients(draws[0], ds)
                model.apply_step(stepped, it)

        snaps.append(_run_phases(T, state, ds, step))
        torch.cuda.synchronize()
    for a, b in zip(snaps[0][1], snaps[1][1]):
        assert np.array_equal(a, b)
