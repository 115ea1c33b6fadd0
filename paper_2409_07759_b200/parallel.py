"""Data parallelism over training views.

One process per GPU.  Every rank holds a replica of the model state and the
same numpy stream, so each iteration all ranks draw the same G (frame, view)
samples; rank r renders sample r.  The only exchange is one allreduce(sum)
of the dense optimization-space gradient buffer (num_gs x 14 float32) before
the replicated, bit-identical fused Adam + SGLD step (Philox counters are
shared, so replicas never diverge).  Generations active in any sampled frame
are stepped (batch-G semantics; G = 1 is exactly the reference).
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


def init_from_env(backend: str = "nccl"):
    """torchrun-style init (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT)."""
    import torch
    import torch.distributed as dist

    if "RANK" not in os.environ or int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return None
    if not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend=backend)
    return DataParallel()
