"""Data-parallel plumbing on CPU with the gloo backend, world_size 2:
identical per-iteration draws on every rank, the union of stepped
generations, and the averaged gradient allreduce."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_07759_b200 import train
        from paper_2409_07759_b200.parallel import DataParallel
        import paper_2409_07759_b200 as P

        dp = DataParallel()
        cfg = train.TrainConfig(swin_size=4, num_gs=40, rng_seed=5)
        state = train.init_state(cfg)
        state.genesis_done = True
        train.schedule_expire(state)
        train.mature(1, state, writer=None)
        res = {}
        for it in range(6):
            draws = train.sample_views(state, 1, 5, [0, 1, 2], dp.world_size)
            stepped = train.stepped_generations(state.slices, [f for f, _ in draws])
            res[it] = (draws, stepped, draws[dp.rank])
        grads = torch.full((8, 14), float(rank + 1))
        dp.allreduce_grads(grads)
        res["grads"] = grads.numpy().copy()
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_two_rank_draws_and_allreduce():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    for it in range(6):
        assert r0[it][0] == r1[it][0]          # every rank draws the same G samples
        assert r0[it][1] == r1[it][1]          # and steps the same generations
        assert r0[it][2] == r0[it][0][0] and r1[it][2] == r1[it][0][1]
        frames = [f for f, _ in r0[it][0]]
        assert any(r0[it][1]) and len(r0[it][1]) == 4
    np.testing.assert_array_equal(r0["grads"], np.full((8, 14), 1.5))
    np.testing.assert_array_equal(r1["grads"], np.full((8, 14), 1.5))
