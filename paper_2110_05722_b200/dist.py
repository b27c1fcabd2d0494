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
     compute stream, finishes the deferred bias/LN column sums into the fp32
     accumulators, sum-reduces the fp32 bucket, narrows the reduced values into
     the fp16 workspace and counts the non-finite ones;
  3. the optimizer runs after the last bucket with an identical skip decision
     on every rank (see the modes below).

The bucket exchange runs in fp32 (the accumulators, narrowed after the sum, as
the reference narrows once after its own sum: F/engine.py:152-157).  Two modes
(`DataParallel(mode=...)`, env LS2_DP_MODE):
  * "shard" (default): each bucket is reduce-scattered, every rank narrows and
    Adam-updates only its 1/N chunk of each bucket (SPEC.md:573 makes the
    element shard legal), the non-finite count is a scalar all-reduce, and the
    updated params16 chunks are all-gathered in place;
  * "allreduce": each bucket is all-reduced and every rank narrows and updates
    the whole workspace.
Buckets start on multiples of `align` = world x 64 elements (the workspace is
padded to one), so every per-rank chunk is equal and 256-byte aligned.

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

    def _span_call(self, fn, t, send_off, recv_off, count, stream):
        from . import _lib
        base = t.data_ptr()
        es = t.element_size()
        code = _lib.I32 if t.dtype == torch.int32 else _lib.dtype_code(t)
        st = stream.cuda_stream if stream is not None else _lib.stream_handle()
        _lib.call(fn, self.handle, base + send_off * es, base + recv_off * es, count, code, st)

    def reduce_scatter(self, t: torch.Tensor, start: int, stop: int, stream=None):
        """In place over t[start:stop]: this rank's chunk of the sum lands at
        start + rank*c (c = (stop - start) / world)."""
        c = (stop - start) // self.world
        self._span_call("ls2_comm_reduce_scatter", t, start, start + self.rank * c, c, stream)

    def all_gather(self, t: torch.Tensor, start: int, stop: int, stream=None):
        """In place over t[start:stop]: every rank's chunk r*c lands everywhere."""
        c = (stop - start) // self.world
        self._span_call("ls2_comm_all_gather", t, start + self.rank * c, start, c, stream)

    def allreduce_i32(self, t: torch.Tensor, stream=None):
        self._span_call("ls2_comm_allreduce", t, 0, 0, t.numel(), stream)

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

    def __init__(self, links, n: int, bucket_elems: int, align: int = 1):
        self.links = sorted(((o, o + ln, nm) for nm, o, ln in links), key=lambda x: x[0])
        self.align = max(1, int(align))
        self.n = int(n)
        self.n_pad = -(-self.n // self.align) * self.align
        self.bucket = max(1, int(bucket_elems))
        self.reset()

    def reset(self):
        self.done: set = set()
        self.idx = len(self.links)         # links[idx:] are finished
        self.frontier = self.n
        self.issued = self.n_pad           # [issued, n_pad) already exchanged

    def _advance(self):
        while self.idx > 0 and self.links[self.idx - 1][2] in self.done:
            self.idx -= 1
            self.frontier = self.links[self.idx][0]

    def _start(self) -> int:
        """Lowest aligned bucket start inside the finished suffix."""
        return -(-self.frontier // self.align) * self.align

    def ready(self, names) -> list:
        self.done.update(names)
        self._advance()
        lo = self._start()
        if self.issued - lo >= self.bucket:
            span = (lo, self.issued)
            self.issued = lo
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


MODES = ("shard", "allreduce")


class DataParallel:
    """Bucketed fp32 gradient exchange + totals all-reduce over the ranks.

    mode "shard": reduce-scatter buckets, Adam on the rank's chunks, all-gather
    params16; "allreduce": all-reduce buckets, every rank updates everything.
    force=True makes a one-rank job take the exchange path too (one-rank NCCL
    communicator), so the overlapped step can be tested on a single GPU."""

    def __init__(self, group=None, bucket_bytes: int = 16 << 20, force: bool = False,
                 mode: str | None = None, native: bool = True):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.bucket_bytes = int(bucket_bytes)
        self.force = bool(force)
        mode = mode or os.environ.get("LS2_DP_MODE", "shard")
        if mode not in MODES:
            raise ValueError(f"data-parallel mode must be one of {MODES}, got {mode!r}")
        self.mode = mode
        # native=False: the collectives go through torch.distributed (e.g. gloo on
        # CUDA tensors, several ranks sharing one GPU in the tests) instead of the
        # NCCL binding; the step then runs eagerly (no CUDA graph)
        self.native = bool(native)
        self.comm: NcclComm | None = None
        self.comm_stream = None

    @property
    def active(self) -> bool:
        return self.world > 1 or self.force

    def setup_device(self, device):
        """Create the native communicator and the comm stream (CUDA only)."""
        if self.active and self.comm is None and self.comm_stream is None:
            if self.native:
                self.comm = NcclComm(self.rank, self.world, device, self.group)
            # default priority: the exchange's kernels take SMs the backward leaves
            # free instead of pre-empting it (measured on one rank: high priority
            # slowed the backward by more than the exchange's own time;
            # LS2_COMM_PRIORITY=high restores it)
            low = os.environ.get("LS2_COMM_PRIORITY", "low") == "low"
            self.comm_stream = torch.cuda.Stream(device=device, priority=0 if low else -100)
        return self

    def buckets(self, n: int, elem_bytes: int = 2):
        """[(start, stop)] over n elements, last bucket first (reverse layout order)."""
        per = max(1, self.bucket_bytes // elem_bytes)
        spans = [(s, min(n, s + per)) for s in range(0, n, per)]
        return list(reversed(spans))

    @property
    def sharded(self) -> bool:
        return self.mode == "shard"

    @property
    def align(self) -> int:
        """Bucket-start granularity in elements: equal, 256-byte aligned chunks."""
        return 64 * (self.world if self.sharded else 1)

    def padded(self, n: int) -> int:
        a = self.align
        return -(-int(n) // a) * a

    def exchange_plan(self, links, n: int, elem_bytes: int = 4) -> GradExchange:
        return GradExchange(links, n, max(1, self.bucket_bytes // elem_bytes), self.align)

    def chunk(self, start: int, stop: int) -> tuple:
        """(offset, length) of this rank's chunk of bucket [start, stop)."""
        if not self.sharded:
            return start, stop - start
        c = (stop - start) // self.world
        return start + self.rank * c, c

    def reduce_scatter_span(self, flat: torch.Tensor, start: int, stop: int, stream=None):
        if self.comm is not None:
            self.comm.reduce_scatter(flat, start, stop, stream=stream)
        elif self.world > 1:
            c = (stop - start) // self.world
            o = start + self.rank * c
            if flat.is_cuda:      # gloo on CUDA tensors: a sum of the whole span, keep our chunk
                dist.all_reduce(flat[start:stop], op=dist.ReduceOp.SUM, group=self.group)
                return
            out = torch.empty(c, dtype=flat.dtype, device=flat.device)
            dist.reduce_scatter_tensor(out, flat[start:stop].contiguous(), op=dist.ReduceOp.SUM,
                                       group=self.group)
            flat[o:o + c].copy_(out)

    def all_gather_span(self, flat: torch.Tensor, start: int, stop: int, stream=None):
        if self.comm is not None:
            self.comm.all_gather(flat, start, stop, stream=stream)
        elif self.world > 1:
            c = (stop - start) // self.world
            o = start + self.rank * c
            if flat.is_cuda:      # gloo on CUDA tensors: everyone else's chunks zeroed, summed
                buf = torch.zeros(stop - start, dtype=flat.dtype, device=flat.device)
                buf[o - start:o - start + c].copy_(flat[o:o + c])
                dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
                flat[start:stop].copy_(buf)
                return
            out = torch.empty(stop - start, dtype=flat.dtype, device=flat.device)
            dist.all_gather_into_tensor(out, flat[o:o + c].contiguous(), group=self.group)
            flat[start:stop].copy_(out)

    def allreduce_count(self, t: torch.Tensor, stream=None):
        """Sum an int32 counter over the ranks (the non-finite gradient count)."""
        if self.comm is not None:
            self.comm.allreduce_i32(t, stream=stream)
        elif self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

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

    def shard_task(self, task):
        """Every rank trains on its own batches: rank r's step s is the wrapped
        task's step s * world + r (a task built from one seed would otherwise
        hand every rank the same batch)."""
        return task if self.world <= 1 else RankShardedTask(task, self.rank, self.world)

    def max_scalar(self, x: float, device=None) -> float:
        if self.world <= 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


class RankShardedTask:
    """Interleaves a (seed, step)-pure task over the ranks: rank r, step s reads
    batch s * world + r.  The union of one step's batches over the ranks is a
    contiguous run of the single-process stream."""

    def __init__(self, task, rank: int, world: int):
        self.task, self.rank, self.world = task, int(rank), int(world)

    def batch(self, step: int):
        return self.task.batch(int(step) * self.world + self.rank)

    def possible_shapes(self):
        return self.task.possible_shapes()

    def __getattr__(self, name):
        return getattr(self.task, name)
