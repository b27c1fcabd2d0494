"""Data-parallel plumbing: one process per GPU, NCCL over NVLink/NVSwitch.

The reference trains single-process and "consumes already-reduced gradients"
(F/engine.py:4-7); LightSeq2 itself used PyTorch's all-reduce
(PAPER.md:1392).  Here each rank runs the identical fused step on its own
batch shard and the exchange is overlapped with the backward pass:

  1. after the criterion: all-reduce (sum) of the totals (loss, token count,
     correct), so the narrow scale is loss_scale / GLOBAL token count on every
     rank (F/engine.py:153);
  2. backward finishes parameters in exactly reverse workspace-layout order
     (dec_ln, dec5..dec0, cross_kv + enc_ln, enc5..enc0, embeddings), so the
     finished part of the flat workspace is always a suffix [frontier, n).
     `GradExchange` turns "these parameters are final" notices into contiguous
     buckets; for each bucket the comm stream waits on an event from the
     compute stream, narrows fp32 accumulators (+ deferred bias/LN column
     sums) into the fp16 workspace, sum-all-reduces it, and counts non-finite
     values of the REDUCED bucket;
  3. the compute stream joins the comm stream once, then runs Adam with an
     identical skip decision on every rank.

Everything is stream-ordered enqueue work, so the whole step — collectives
included — is captured in the bucket's CUDA graph.  On CUDA the collectives
go through the native NCCL binding (`NcclComm`, ls2_comm_*); the same
planner drives torch.distributed (gloo) on CPU tensors in the tests.
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


def _nccl_lib_path():
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        p = os.path.join(base, "lib", "libnccl.so.2")
        return p if os.path.exists(p) else None
    except Exception:
        return None


class NcclComm:
    """A native NCCL communicator over the ranks of `group` (ls2_comm_*).

    Rank 0 draws the ncclUniqueId; it is shared through torch.distributed
    (any backend).  world == 1 gives a one-rank communicator — the same code
    path, used by the single-GPU tests of the overlapped, graph-captured step.
    """

    def __init__(self, rank: int, world: int, device, group=None):
        import ctypes
        from . import _lib
        lib = _lib.load_library()
        path = _nccl_lib_path()
        _lib.call("ls2_comm_load", path.encode() if path else None)
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _lib.call("ls2_comm_unique_id", ctypes.addressof(uid))
        if world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            ctypes.memmove(uid, box[0], 128)
        h = ctypes.c_void_p()
        dev = torch.device(device)
        _lib.call("ls2_comm_init", ctypes.byref(h), world, rank, ctypes.addressof(uid),
                  dev.index or 0)
        self.handle = h.value
        self.rank, self.world = rank, world
        self._lib = lib

    def allreduce(self, t: torch.Tensor, start: int = 0, stop: int | None = None, stream=None):
        from . import _lib
        stop = t.numel() if stop is None else stop
        base = t.data_ptr() + start * t.element_size()
        st = stream.cuda_stream if stream is not None else _lib.stream_handle()
        _lib.call("ls2_comm_allreduce", self.handle, base, base, stop - start,
                  _lib.dtype_code(t), st)

    def close(self):
        if self.handle:
            from . import _lib
            _lib.call("ls2_comm_destroy", self.handle)
            self.handle = None


class GradExchange:
    """Turns "parameters final" notices into contiguous reverse-order buckets.

    links: (name, offset, length) of the flat workspace.  Backward finishes a
    suffix of the layout at a time; `ready(names)` records finished names,
    advances the frontier over the finished suffix and returns the spans
    [start, stop) to exchange now: one span once at least `bucket_elems`
    elements are pending, everything pending on `flush()`.
    """

    def __init__(self, links, n: int, bucket_elems: int):
        self.links = sorted(((o, o + ln, nm) for nm, o, ln in links), key=lambda x: x[0])
        self.n = int(n)
        self.bucket = max(1, int(bucket_elems))
        self.reset()

    def reset(self):
        self.done: set = set()
        self.idx = len(self.links)         # links[idx:] are finished
        self.frontier = self.n
        self.issued = self.n               # [issued, n) already exchanged

    def _advance(self):
        while self.idx > 0 and self.links[self.idx - 1][2] in self.done:
            self.idx -= 1
            self.frontier = self.links[self.idx][0]

    def ready(self, names) -> list:
        self.done.update(names)
        self._advance()
        if self.issued - self.frontier >= self.bucket:
            span = (self.frontier, self.issued)
            self.issued = self.frontier
            return [span]
        return []

    def finish_all(self) -> list:
        """Every parameter is final (end of backward): exchange the rest."""
        self.done.update(nm for _, _, nm in self.links)
        return self.flush()

    def flush(self) -> list:
        self._advance()
        if self.frontier != 0:
            missing = [nm for _, _, nm in self.links[:self.idx]]
            raise RuntimeError(f"gradient exchange: parameters never finished: {missing[:4]}")
        if self.issued > 0:
            span = (0, self.issued)
            self.issued = 0
            return [span]
        return []


class DataParallel:
    """Bucketed gradient all-reduce + totals all-reduce over the ranks.

    force=True makes a one-rank job take the exchange path too (one-rank NCCL
    communicator), so the overlapped step can be tested on a single GPU."""

    def __init__(self, group=None, bucket_bytes: int = 8 << 20, force: bool = False):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.bucket_bytes = int(bucket_bytes)
        self.force = bool(force)
        self.comm: NcclComm | None = None
        self.comm_stream = None

    @property
    def active(self) -> bool:
        return self.world > 1 or self.force

    def setup_device(self, device):
        """Create the native communicator and the comm stream (CUDA only)."""
        if self.active and self.comm is None:
            self.comm = NcclComm(self.rank, self.world, device, self.group)
            self.comm_stream = torch.cuda.Stream(device=device, priority=-100)
        return self

    def buckets(self, n: int, elem_bytes: int = 2):
        """[(start, stop)] over n elements, last bucket first (reverse layout order)."""
        per = max(1, self.bucket_bytes // elem_bytes)
        spans = [(s, min(n, s + per)) for s in range(0, n, per)]
        return list(reversed(spans))

    def exchange_plan(self, links, n: int, elem_bytes: int = 2) -> GradExchange:
        return GradExchange(links, n, max(1, self.bucket_bytes // elem_bytes))

    def allreduce_totals(self, out3: torch.Tensor, stream=None):
        if self.comm is not None:
            self.comm.allreduce(out3, stream=stream)
        elif self.world > 1:
            dist.all_reduce(out3, op=dist.ReduceOp.SUM, group=self.group)
        return out3

    def allreduce_span(self, flat: torch.Tensor, start: int, stop: int, stream=None):
        if self.comm is not None:
            self.comm.allreduce(flat, start, stop, stream=stream)
        elif self.world > 1:
            dist.all_reduce(flat[start:stop], op=dist.ReduceOp.SUM, group=self.group)

    def allreduce_grads(self, flat: torch.Tensor):
        """Sum the flat gradient workspace across ranks, bucket by bucket."""
        if not self.active:
            return flat
        for s, e in self.buckets(flat.numel(), flat.element_size()):
            self.allreduce_span(flat, s, e)
        return flat

    def barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)

    def max_scalar(self, x: float, device=None) -> float:
        if self.world <= 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())
