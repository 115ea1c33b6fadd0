"""Data parallelism over training views.

One process per GPU.  Every rank holds a replica of the model state and the
same numpy stream, so each iteration all ranks draw the same G (frame, view)
samples; rank r renders sample r.  The only exchange is one allreduce of the
dense optimization-space gradient buffer (num_gs x 14 float32) before the
replicated, bit-identical fused Adam + SGLD step (Philox counters are
shared, so replicas never diverge; tests/test_gpu_dp.py checks bit equality
of the replicas and of a single-process emulation at world 2).  Generations
active in any sampled frame are stepped (batch-G semantics; G = 1 is exactly
the reference).

Mean, not sum: the reduced gradient is the MEAN over the G views (NCCL AVG;
gloo SUM then x 1/G).  The batch loss is then the mean of the per-view
reference losses, so the gradient keeps the single-view magnitude the
reference's constants were tuned for -- the gamma^w mean-gradient damping,
the regularizer weights (added once, inside the fused step, over the
stepped rows) and Adam's eps = 1e-15 regime see the same scale at every G --
and G = 1 is the reference step bit for bit.  (Adam itself is invariant to
a constant gradient scale; SGD, a config option, is not, and with a sum its
effective learning rate would grow with G.)
"""

from __future__ import annotations

import os


class DataParallel:
    def __init__(self, group=None, average: bool = True):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world_size = dist.get_world_size(group)
        self.average = average

    def allreduce_grads(self, grads) -> None:
        if self.world_size == 1:
            return
        if self.average and self.dist.get_backend(self.group) == "nccl":
            # NCCL averages in the collective (no separate scaling pass)
            self.dist.all_reduce(grads, op=self.dist.ReduceOp.AVG, group=self.group)
            return
        self.dist.all_reduce(grads, op=self.dist.ReduceOp.SUM, group=self.group)
        if self.average:
            grads.mul_(1.0 / self.world_size)

    def barrier(self):
        self.dist.barrier(group=self.group)


def local_device_index() -> int:
    """This rank's GPU: LOCAL_RANK, wrapped onto the visible devices (so a
    world-2 gloo run can share one GPU for testing)."""
    import torch

    n = max(torch.cuda.device_count(), 1)
    return int(os.environ.get("LOCAL_RANK", "0")) % n


def init_from_env(backend: str = "nccl"):
    """torchrun-style init (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT).
    SS_DP_BACKEND overrides the backend (e.g. "gloo" to run two ranks on one
    GPU, which NCCL refuses)."""
    import torch
    import torch.distributed as dist

    if "RANK" not in os.environ or int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return None
    backend = os.environ.get("SS_DP_BACKEND", backend)
    if not dist.is_initialized():
        if torch.cuda.is_available():
            torch.cuda.set_device(local_device_index())
        dist.init_process_group(backend=backend)
    return DataParallel()
