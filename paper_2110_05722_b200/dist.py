"""Data-parallel plumbing: one process per GPU, NCCL over NVLink/NVSwitch.

The reference trains single-process and "consumes already-reduced gradients"
(F/engine.py:4-7); LightSeq2 itself used PyTorch's all-reduce
(PAPER.md:1392).  Here each rank runs the identical fused step on its own
batch shard, then:

  1. all-reduce (sum) of the criterion totals (loss, token count, correct) so
     the gradient scale is loss_scale / GLOBAL token count on every rank;
  2. narrow to the fp16 gradient workspace with that scale;
  3. all-reduce (sum) of the flat fp16 workspace in contiguous buckets, in
     reverse layout order (the tail of the workspace — last layers — is
     finished first by backward), on the compute stream;
  4. non-finite count on the REDUCED gradients -> identical skip decision on
     every rank -> workspace Adam.

Device-agnostic: the same class drives gloo on CPU tensors in the tests.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def init_from_env(backend: str | None = None):
    """torchrun-style init (RANK/WORLD_SIZE/MASTER_*); returns (rank, world, local_rank)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return rank, world, local


class DataParallel:
    """Bucketed fp16 gradient all-reduce + scalar totals all-reduce."""

    def __init__(self, group=None, bucket_bytes: int = 32 << 20):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.bucket_bytes = int(bucket_bytes)

    @property
    def active(self) -> bool:
        return self.world > 1

    def buckets(self, n: int, elem_bytes: int = 2):
        """[(start, stop)] over n elements, last bucket first (reverse layout order)."""
        per = max(1, self.bucket_bytes // elem_bytes)
        spans = [(s, min(n, s + per)) for s in range(0, n, per)]
        return list(reversed(spans))

    def allreduce_totals(self, out3: torch.Tensor):
        if self.active:
            dist.all_reduce(out3, op=dist.ReduceOp.SUM, group=self.group)
        return out3

    def allreduce_grads(self, flat: torch.Tensor):
        """Sum the flat gradient workspace across ranks, bucket by bucket."""
        if not self.active:
            return flat
        for s, e in self.buckets(flat.numel(), flat.element_size()):
            dist.all_reduce(flat[s:e], op=dist.ReduceOp.SUM, group=self.group)
        return flat

    def barrier(self):
        if self.active:
            dist.barrier(group=self.group)

    def max_scalar(self, x: float, device=None) -> float:
        if not self.active:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())
