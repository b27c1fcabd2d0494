"""Training driver (F/engine.py): fused forward/backward on the planned device
arena, scale+narrow into the fp16 workspace, (data-parallel all-reduce), one
workspace optimizer pass — captured as ONE CUDA graph per (mode, B, L) bucket.

Per step the host only: builds the batch (numpy), writes it and the per-step
dropout seeds into pinned staging buffers, replays the bucket's graph (which
begins with the H2D copies and ends with a D2H copy of loss / token count /
correct / applied-flag / non-finite count) and reads those five numbers.
Skip decisions (non-finite loss or gradient) and the Adam step counter live
on the device, so a skipped step needs no extra host round trip.
"""

from __future__ import annotations

import ctypes
import gc
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import checkpoint as ckpt
from .config import RunConfig
from .data import make_task
from .dist import DataParallel
from .errors import DataError
from .memplan import PlannedArena, RecordingArena, TensorTag, classify, estimate_capacity
from .model import Batch, MaskBank, SeedTable, Transformer, _ViewSink, make_model, validate_batch
from .trainer import OptimConfig, Workspace, _state, bias_correction_rows, workspace_pack

EVAL_STEP_BASE = 1 << 30


class _no_gc:
    """Collect garbage first, then keep the collector off while a CUDA graph is
    being captured: destroying another (dead) graph mid-capture invalidates it."""

    def __enter__(self):
        torch.cuda.synchronize()
        gc.collect()
        self._was = gc.isenabled()
        gc.disable()

    def __exit__(self, *a):
        if self._was:
            gc.enable()
        torch.cuda.synchronize()


@dataclass
class StepMetrics:
    step: int
    loss: float
    tokens: int
    accuracy: float
    tokens_per_sec: float
    arena_high_water: int
    skipped: bool
    nonfinite: int

    def as_dict(self) -> dict:
        return dict(self.__dict__)


class _StaticIO:
    """Device batch buffers of one bucket shape + their pinned host twins."""

    def __init__(self, b: int, l: int, device):
        pin = lambda *s: torch.zeros(*s, dtype=torch.int64).pin_memory()  # noqa: E731
        self.h_src, self.h_tin, self.h_tout, self.h_len = pin(b, l), pin(b, l), pin(b, l), pin(b)
        self.src = torch.zeros((b, l), dtype=torch.int64, device=device)
        self.tin = torch.zeros_like(self.src)
        self.tout = torch.zeros_like(self.src)
        self.len = torch.zeros(b, dtype=torch.int64, device=device)
        self.pad_id = 0

    def stage(self, batch: Batch):
        self.h_src.copy_(torch.from_numpy(np.asarray(batch.src, dtype=np.int64)))
        self.h_tin.copy_(torch.from_numpy(np.asarray(batch.tgt_in, dtype=np.int64)))
        self.h_tout.copy_(torch.from_numpy(np.asarray(batch.tgt_out, dtype=np.int64)))
        self.h_len.copy_(torch.from_numpy(np.asarray(batch.src_len, dtype=np.int64)))
        self.pad_id = int(batch.pad_id)

    def upload(self):
        for d, h in ((self.src, self.h_src), (self.tin, self.h_tin), (self.tout, self.h_tout),
                     (self.len, self.h_len)):
            d.copy_(h, non_blocking=True)

    def spans(self) -> list:
        """(dst, src, nbytes) of the batch's H2D copies."""
        return [(d.data_ptr(), h.data_ptr(), 8 * d.numel())
                for d, h in ((self.src, self.h_src), (self.tin, self.h_tin),
                             (self.tout, self.h_tout), (self.len, self.h_len))]

    def batch(self) -> Batch:
        return Batch(self.src, self.tin, self.tout, self.len, self.pad_id)

    @property
    def h2d_bytes(self) -> int:
        return 8 * (3 * self.src.numel() + self.len.numel())


class TrainingEngine:
    def __init__(self, run_cfg: RunConfig, task=None, dp: DataParallel | None = None,
                 device=None):
        self.cfg = run_cfg
        ctx = _lib.context(device)
        self.device = ctx.device
        self.model = make_model(run_cfg.model)
        self.dp = dp if dp is not None else DataParallel()
        # under data parallelism every rank reads its own batches (dist.RankShardedTask)
        self.task = task if task is not None else self.dp.shard_task(make_task(run_cfg))
        t = run_cfg.train
        self.optim = OptimConfig(algorithm=t.algorithm, lr=t.lr, beta1=t.beta1, beta2=t.beta2,
                                 eps_opt=t.eps_opt, weight_decay=t.weight_decay,
                                 momentum=t.momentum, loss_scale=t.loss_scale)
        init = self.model.init_params(t.seed)
        self.ws: Workspace = workspace_pack([(n, init[n]) for n in self.model.param_names],
                                            t.algorithm)
        del init
        n = self.ws.n_elements
        # the exchange's buckets split into equal aligned per-rank chunks: pad the
        # workspace storage (never the [0, n) views) to the planner's granularity
        n_pad = self.dp.padded(n) if self.dp.active else n
        self.ws.pad_storage(n_pad)
        self.pviews = self.ws.param_views()
        self.grad_acc = torch.zeros(n_pad, dtype=torch.float32, device=self.device)
        self.gviews = {lk.name: self.grad_acc[lk.offset:lk.offset + lk.length].view(lk.shape)
                       for lk in self.ws.links}
        self._opt = _state(self.ws, self.optim)
        self._applied_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._nonfinite = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._dev_out = torch.zeros(5, dtype=torch.float64, device=self.device)
        self._host_out = torch.zeros(5, dtype=torch.float64).pin_memory()
        # the step's metrics reach the host BEFORE the optimizer runs (they are known
        # once the non-finite count is): train_step waits on this event, not on the
        # stream, so the host returns and enqueues the next step while Adam (and the
        # next step's mask draw) still run; the next replay is stream-ordered after
        # them.  Data parallelism keeps the end-of-step copy.
        self._metrics_ev = torch.cuda.Event(external=True)
        self._early_report = os.environ.get("LS2_EARLY_REPORT", "1") != "0"
        self._one_copy = os.environ.get("LS2_COPY_SPANS", "1") != "0"
        self._xplan = None
        self._span_tables: dict = {}
        self.merge_spans = True          # tests set False to run the per-chunk update on 1 rank
        if self.dp.active:
            self.dp.setup_device(self.device)
            self._xplan = self.dp.exchange_plan(
                [(lk.name, lk.offset, lk.length) for lk in self.ws.links], n)
        self.applied_steps = 0
        self.skip_count = 0
        self.arena: PlannedArena | None = None
        self.capacity = 0
        self._io: dict = {}
        self._graphs: dict = {}
        self._launches: dict = {}
        self._finish_tables: dict = {}
        self.use_graphs = bool(t.cuda_graphs)
        # weight-gradient GEMMs on a low-priority side lane (LS2_WGRAD_LANE=1).  Off
        # by default: measured 1% slower at T-base, because the one-wave fused
        # kernels cannot co-reside with a concurrent GEMM's CTAs
        self.use_lane = os.environ.get("LS2_WGRAD_LANE", "0") == "1"
        # weight-gradient GEMMs batched across layers (model._WgradBatch):
        # LS2_WGRAD_BATCH=0 off, =k flush every k layers, =end once at the end of
        # backward; default: at the end, every 2 layers under data parallelism
        # (so the bucket exchange still overlaps the rest of backward)
        wb = os.environ.get("LS2_WGRAD_BATCH", "auto")
        self.wgrad_group = None if wb == "0" else 0 if wb == "end" else \
            ((2 if self.dp.active else 0) if wb == "auto" else int(wb))
        # every forward dropout site of a step drawn by one launch (model.MaskBank)
        self.masks = MaskBank(self.device) if os.environ.get("LS2_MASK_BANK", "1") != "0" else None
        # next step's site seeds: the bank draws step t+1's bits beside step t's Adam
        self._seeds_next = SeedTable(self.device)
        # LS2_EARLY_MASKS=1: draw the next step's bits layer by layer during backward
        #   =opt (default): the whole bank at once beside this step's narrow pass and
        #   optimizer (HBM-bound), capped at one CTA per SM so both share every SM;
        #   =0: in-step draw only
        self._early_mode = os.environ.get("LS2_EARLY_MASKS", "opt")
        self._early_masks = self._early_mode in ("1", "opt")
        # host/device overlap: once a step's inputs are on the device (an event
        # recorded inside the graph), the host stages the next step's batch and
        # seeds while the device still runs this one (LS2_OVERLAP_HOST=0: off)
        self._consumed = torch.cuda.Event(external=True)
        self._overlap_host = os.environ.get("LS2_OVERLAP_HOST", "1") != "0"
        self._pre = None                   # (step, batch, key, error) staged ahead
        self.last_out3 = None

    # -- arena setup (F/engine.py:89-103) ----------------------------------------------

    def _dummy_batch(self, b: int, l: int) -> Batch:
        filler = (self.cfg.data.pad_id + 2) % self.cfg.model.vocab
        tok = np.full((b, l), filler, dtype=np.int64)
        return Batch(src=tok, tgt_in=tok.copy(), tgt_out=tok.copy(),
                     src_len=np.full(b, l, dtype=np.int64), pad_id=self.cfg.data.pad_id)

    def _record_shape(self, batch: Batch, compute_grads: bool):
        rec = RecordingArena(self.device)
        sink = _ViewSink(self.gviews, defer=True, lane=self.use_lane,
                         wgrad_group=self.wgrad_group) if compute_grads else None
        self.model.forward_backward(self.pviews, batch,
                                    p_drop=self.cfg.train.p_drop if compute_grads else 0.0,
                                    alpha=self.cfg.train.alpha, seed=self.cfg.train.seed,
                                    step=0, arena=rec, sink=sink, compute_grads=compute_grads,
                                    masks=self.masks)
        return rec.finish()

    def setup_arena(self) -> int:
        """Dry-run every bucket shape, size the arena once (bytes), register plans."""
        recorded = {}
        if self.masks is not None:
            shapes = list(self.task.possible_shapes())
            mt = max(b * l for b, l in shapes)
            self.masks.configure(mt, mt)
        for b, l in self.task.possible_shapes():
            batch = self._dummy_batch(b, l)
            recorded[("train", b, l)] = self._record_shape(batch, True)
            recorded[("eval", b, l)] = self._record_shape(batch, False)
        torch.cuda.synchronize()
        self.capacity = estimate_capacity(recorded.values())
        self.arena = PlannedArena(self.capacity, self.device)
        for key, lts in recorded.items():
            self.arena.register_plan(key, lts)
        torch.cuda.empty_cache()
        return self.capacity

    def memory_report(self) -> dict:
        tags = [TensorTag("params16", "parameter"), TensorTag("grads16", "gradient"),
                TensorTag("grad_acc32", "gradient"), TensorTag("moments", "moment"),
                TensorTag("arena", "intermediate")]
        p = self.ws.n_elements
        return {"classes": classify(tags), "parameters": p,
                "permanent_bytes": self.ws.state_bytes() + p * 4,
                "temporary_capacity_bytes": self.capacity}

    # -- the device step -------------------------------------------------------------

    def _io_for(self, b, l) -> _StaticIO:
        io = self._io.get((b, l))
        if io is None:
            io = self._io[(b, l)] = _StaticIO(b, l, self.device)
        return io

    def _stage_next_seeds(self, step: int):
        """Host: the site seeds of step+1 into the next-step table's staging buffer."""
        t = self.cfg.train
        self.model.register_seeds(self._seeds_next, t.seed, step + 1, t.p_drop)
        self._seeds_next.write_host(sync=False)

    def _fwd_bwd(self, io: _StaticIO, key, step: int, upload: bool = True):
        t = self.cfg.train
        if upload:
            # every host->device input of the step first: the batch, this step's
            # site seeds, (the next step's seeds); then mark them consumed so the
            # host can stage the next step while this one runs (train_step)
            # all of them as ONE kernel reading the pinned buffers (ls2_copy_spans)
            # instead of one copy-engine node each (LS2_COPY_SPANS=0: the copies)
            spans = io.spans()
            seeds = None
            if t.p_drop > 0.0:
                seeds = self.model.seed_table(self.device)
                self.model.register_seeds(seeds, t.seed, step, t.p_drop)
                spans.append(seeds.stage_span())
            if self.masks is not None and self._early_masks and t.p_drop > 0.0:
                if not torch.cuda.is_current_stream_capturing():
                    self._stage_next_seeds(step)
                nx = self._seeds_next
                spans.append((nx.dev.data_ptr(), nx.host.data_ptr(), 8 * len(nx.values)))
            if self._one_copy:
                n = len(spans)
                _lib.call("ls2_copy_spans", (ctypes.c_void_p * n)(*[s[0] for s in spans]),
                          (ctypes.c_void_p * n)(*[s[1] for s in spans]),
                          (ctypes.c_int64 * n)(*[s[2] for s in spans]), n, _lib.stream_handle())
            else:
                io.upload()
                for tab in ([seeds] if seeds is not None else []) + \
                        ([self._seeds_next] if len(spans) > 4 + (seeds is not None) else []):
                    n = len(tab.values)
                    tab.dev[:n].copy_(tab.host[:n], non_blocking=True)
            if seeds is not None:
                seeds.uploaded()
            self._consumed.record()
        self.arena.begin(key)
        sink = _ViewSink(self.gviews, defer=True, lane=self.use_lane, wgrad_group=self.wgrad_group)
        self._bank_done = None
        if self.masks is not None and self._early_masks and t.p_drop > 0.0:
            # the next step's dropout bits, layer by layer as backward releases them
            self._bank_table = self._seeds_next if upload else self.model.seed_table(self.device)
            if self._early_mode == "1":
                sink.on_layer_done = self._bank_layer_done
        if self.dp.active:
            # buckets are narrowed / all-reduced on the comm stream while the
            # backward pass is still running (dist.py)
            self._nonfinite.zero_()
            self._xplan.reset()
            self._totals_sent = False
            self._deferred_done = set()
            self._buckets, self._shard_spans = [], []
            sink.on_ready = lambda names, _s=sink: self._on_ready(_s, names)
        out = self.model.forward_backward(
            self.pviews, io.batch(), p_drop=t.p_drop, alpha=t.alpha, seed=t.seed, step=step,
            arena=self.arena, sink=sink, grad_scale=float(t.act_grad_scale), validate=False,
            upload_seeds=False, masks=self.masks)
        self.arena.end()
        return out.out3, sink

    def capture_device_graph(self, key):
        """Graph of one step with device-resident inputs (no H2D/D2H): the
        benchmark's `value` path.  Also records how many libls2 kernels a step
        launches (cuBLAS kernels not counted)."""
        b, l = key[1], key[2]
        io = self._io_for(b, l)
        g = torch.cuda.CUDAGraph()
        n0 = _lib.launches()
        with _no_gc():
            with torch.cuda.graph(g, stream=_lib.context().compute_stream, **self._capture_kw()):
                out3, sink = self._fwd_bwd(io, key, 0, upload=False)
                self._update(out3, sink, host_copy=False)
        self._launches[key] = _lib.launches() - n0
        torch.cuda.synchronize()
        return g

    def _capture_kw(self) -> dict:
        # NCCL's proxy thread may touch the CUDA API while our stream captures
        return {"capture_error_mode": "thread_local"} if self.dp.active else {}

    def launches_per_step(self, key) -> int:
        return int(self._launches.get(key, 0))

    def device_step(self, key, step: int):
        """One eager step on already-resident inputs (DP fallback for timing)."""
        io = self._io_for(key[1], key[2])
        n0 = _lib.launches()
        self._update(*self._fwd_bwd(io, key, step, upload=False), host_copy=False)
        self._launches[key] = _lib.launches() - n0

    # -- data-parallel exchange overlapped with backward (dist.py) ----------------------

    def _on_ready(self, sink, names):
        spans = self._xplan.finish_all() if names is None else self._xplan.ready(names)
        for span in spans:
            self._exchange_bucket(sink, *span)

    def _exchange_bucket(self, sink, start: int, stop: int):
        """On the comm stream, after everything the compute stream has enqueued so
        far: finish the deferred column sums that reach into [start, stop) into the
        fp32 accumulators, sum-reduce the fp32 bucket (reduce-scatter: this rank's
        chunk; all-reduce: all of it), narrow the reduced values into grads16 and
        count the non-finite ones (dist.py)."""
        t = self.cfg.train
        dp = self.dp
        cs = dp.comm_stream
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        cs.wait_event(ev)
        with torch.cuda.stream(cs):
            out3 = sink.totals
            if not self._totals_sent:
                dp.allreduce_totals(out3, stream=cs)
                self._totals_sent = True
            ws = self.ws
            entries = []
            for e in sink.deferred:
                if e[0] in self._deferred_done:
                    continue
                off, ln = ws.resolve(e[0])
                if off + ln > start:           # finished: it lies in the finished suffix
                    entries.append(e)
                    self._deferred_done.add(e[0])
            if entries:
                tab = self._finish_table(entries)
                _lib.call("ls2_finish_acc32", tab[0].data_ptr(), tab[1].data_ptr(), tab[2], None,
                          self.grad_acc.data_ptr(), cs.cuda_stream)
            if dp.sharded:
                dp.reduce_scatter_span(self.grad_acc, start, stop, stream=cs)
            else:
                dp.allreduce_span(self.grad_acc, start, stop, stream=cs)
            off, c = dp.chunk(start, stop)
            _lib.call("ls2_scale_narrow", self.grad_acc.data_ptr() + 4 * off,
                      ws.grads16.data_ptr() + 2 * off, c, float(t.loss_scale),
                      out3.data_ptr(), -1, float(1.0 / t.act_grad_scale),
                      self._nonfinite.data_ptr(), cs.cuda_stream)
            self._buckets.append((start, stop))
            self._shard_spans.append((off, c))

    def _spans_table(self, spans):
        """(device table, count, longest) of the rank's chunks cut into pieces of
        near-equal length, one CTA each: the chunks differ in size (the last
        bucket holds the whole token table), and one grid row per chunk would
        leave most CTAs idle while the largest chunk finishes."""
        key = tuple(spans)
        hit = self._span_tables.get(key)
        if hit is None:
            total = sum(c for _, c in spans)
            piece = max(2048, -(-total // (148 * 8) // 2048) * 2048)
            rows = [(o + k, min(piece, c - k)) for o, c in spans for k in range(0, c, piece)]
            tab = torch.tensor([x for sp in rows for x in sp], dtype=torch.int64,
                               device=self.device)
            hit = self._span_tables[key] = (tab, len(rows), piece)
        return hit

    def _dp_update(self, loss_ptr):
        """Data-parallel optimizer step on the comm stream, after the last bucket.
        shard: global non-finite count (scalar all-reduce), Adam/SGD on this rank's
        chunks, in-place all-gather of the updated params16 chunks; allreduce:
        every rank holds the whole reduced gradient and updates everything."""
        dp, ws, cs = self.dp, self.ws, self.dp.comm_stream
        with torch.cuda.stream(cs):
            st = cs.cuda_stream
            if not dp.sharded:
                self._optimizer(0, ws.n_elements, loss_ptr, st)
                return
            dp.allreduce_count(self._nonfinite, stream=cs)
            spans = []
            for off, c in sorted(sp for sp in self._shard_spans if sp[1] > 0):
                if spans and spans[-1][0] + spans[-1][1] == off:      # adjacent (world 1)
                    spans[-1] = (spans[-1][0], spans[-1][1] + c)
                else:
                    spans.append((off, c))
            if len(spans) == 1 and self.merge_spans:                  # one contiguous range
                self._optimizer(spans[0][0], spans[0][1], loss_ptr, st)
                spans = []
            if not spans:
                pass
            elif self.optim.algorithm == "adam":
                tab, npieces, piece = self._spans_table(spans)
                _lib.call("ls2_adam_spans", ws.params16.data_ptr(), ws.grads16.data_ptr(),
                          ws.m32.data_ptr(), ws.v32.data_ptr(), tab.data_ptr(), npieces, piece,
                          self._opt.hyper.data_ptr(),
                          self._opt.bc.data_ptr(), bias_correction_rows(self._opt.bc), 0,
                          self._applied_dev.data_ptr(), self._nonfinite.data_ptr(), loss_ptr, st)
            else:
                for off, c in spans:
                    self._optimizer(off, c, loss_ptr, st)
            for start, stop in self._buckets:
                dp.all_gather_span(ws.params16, start, stop, stream=cs)

    def _optimizer(self, off: int, n: int, loss_ptr, st):
        ws = self.ws
        if self.optim.algorithm == "adam":
            _lib.call("ls2_adam", ws.params16.data_ptr() + 2 * off,
                      ws.grads16.data_ptr() + 2 * off, ws.m32.data_ptr() + 4 * off,
                      ws.v32.data_ptr() + 4 * off, n, self._opt.hyper.data_ptr(),
                      self._opt.bc.data_ptr(), bias_correction_rows(self._opt.bc), 0,
                      self._applied_dev.data_ptr(), self._nonfinite.data_ptr(), loss_ptr, st)
        else:
            _lib.call("ls2_sgd", ws.params16.data_ptr() + 2 * off,
                      ws.grads16.data_ptr() + 2 * off, ws.m32.data_ptr() + 4 * off, n,
                      self._opt.hyper.data_ptr(), self._nonfinite.data_ptr(), loss_ptr, st)

    _BANK_GROUPS = {"cross_kv.": "tgt"}

    def _bank_layer_done(self, prefixes):
        """Backward released these layers' dropout bits: redraw them for the next
        step on the low-priority side stream, overlapping the rest of backward."""
        bank = self.masks
        if bank.desc is None:
            return
        if prefixes is None:
            groups = ["src"]
        else:
            groups = []
            for p in prefixes:
                g = self._BANK_GROUPS.get(p, p.rstrip("."))
                if g in bank.groups:
                    groups.append(g)
        if not groups:
            return
        side = _lib.context().side_stream
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        side.wait_event(ev)
        with torch.cuda.stream(side):
            for g in groups:
                bank.generate_group(g, self._bank_table.dev)
            if prefixes is None:
                bank.stamp.copy_(self._bank_table.step_slot())
        if prefixes is None:
            self._bank_done = torch.cuda.Event()
            self._bank_done.record(side)

    def _draw_next_bank(self):
        """The next step's dropout bits on the side stream, beside this step's
        narrow pass and optimizer: those are HBM-bound and the draw is integer-ALU
        bound, so with the draw capped at one CTA per SM the two share every SM
        (alone: Adam 236 us + draw 167 us; together 274 us,
        profiles/r3d_overlap.jsonl).  Every read of this step's bits is enqueued
        before this point; the next step finds the stamp and skips its draw."""
        bank = self.masks
        side = _lib.context().side_stream
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        side.wait_event(ev)
        with torch.cuda.stream(side):
            bank.generate(self._bank_table.dev, ctas_per_sm=1)
            bank.stamp.copy_(self._bank_table.step_slot())
        self._bank_done = torch.cuda.Event()
        self._bank_done.record(side)

    def _finish_deferred(self, sink, out3, nonfinite_ptr, entries=None):
        """One launch finishing every deferred bias / LayerNorm gradient (partials
        left by their producers) straight into the fp16 workspace."""
        entries = sink.deferred if (entries is None and sink is not None) else entries
        if not entries:
            return
        tab = self._finish_table(entries)
        t = self.cfg.train
        _lib.call("ls2_finish_narrow", tab[0].data_ptr(), tab[1].data_ptr(), tab[2], None,
                  self.ws.grads16.data_ptr(), float(t.loss_scale), out3.data_ptr(), -1,
                  float(1.0 / t.act_grad_scale), nonfinite_ptr, _lib.stream_handle())

    def _finish_table(self, entries):
        """(desc, chunks, n_chunks) device tables of the deferred entries (cached)."""
        key = tuple((n, buf.data_ptr(), nb, st, k, c) for n, buf, nb, st, k, c in entries)
        tab = self._finish_tables.get(key)
        if tab is None:
            desc, chunks = [], []
            for i, (n, ptr, nb, st, k, c) in enumerate(key):
                off, _ = self.ws.resolve(n)
                desc.append([off, c, ptr // 8, nb, st, k])
                chunks += [(i, c0) for c0 in range(0, c, 64)]
            tab = (torch.tensor(desc, dtype=torch.int64, device=self.device),
                   torch.tensor(chunks, dtype=torch.int32, device=self.device), len(chunks))
            self._finish_tables[key] = tab
        return tab

    def _update(self, out3: torch.Tensor, sink=None, host_copy: bool = True):
        """narrow(+scale) -> [all-reduce] -> non-finite count -> Adam/SGD -> commit."""
        st = _lib.stream_handle()
        t = self.cfg.train
        ws = self.ws
        loss_ptr = out3.data_ptr()
        if self._early_mode == "opt" and self.masks is not None and \
                self.masks.desc is not None and t.p_drop > 0.0 and sink is not None:
            self._draw_next_bank()
        joined = getattr(self, "_bank_done", None)
        reported = False
        if self.dp.active:
            # every bucket was reduced + narrowed + checked on the comm stream;
            # the optimizer (sharded or whole) follows there, then the join
            self._dp_update(loss_ptr)
            ev = torch.cuda.Event()
            ev.record(self.dp.comm_stream)
            torch.cuda.current_stream().wait_event(ev)
        else:
            self._nonfinite.zero_()
            _lib.call("ls2_scale_narrow", self.grad_acc.data_ptr(), ws.grads16.data_ptr(),
                      ws.n_elements, float(t.loss_scale), out3.data_ptr(), -1,
                      float(1.0 / t.act_grad_scale), self._nonfinite.data_ptr(), st)
            self._finish_deferred(sink, out3, self._nonfinite.data_ptr())
            if host_copy and self._early_report:
                # the metrics are final here (the skip decision needs only the
                # non-finite count and the loss): report them before the update
                # written by the report kernel straight into the pinned host
                # buffer (UVA): no D2H copy node ahead of the optimizer
                _lib.call("ls2_step_report", None, self._nonfinite.data_ptr(), loss_ptr,
                          self._host_out.data_ptr(), st)
                self._metrics_ev.record()
                reported = True
            self._optimizer(0, ws.n_elements, loss_ptr, st)
        _lib.call("ls2_step_report", self._applied_dev.data_ptr(), self._nonfinite.data_ptr(),
                  loss_ptr, self._dev_out.data_ptr(), st)
        if joined is not None:
            torch.cuda.current_stream().wait_event(joined)
        if host_copy and not reported:
            self._host_out.copy_(self._dev_out, non_blocking=True)
            self._metrics_ev.record()

    def _run(self, io, key, step, graphed: bool):
        if graphed:
            g = self._graphs.get(key)
            if g is not None:
                g.replay()
                return
        out3, sink = self._fwd_bwd(io, key, step)
        self.last_out3 = out3
        self._update(out3, sink)

    def _capture(self, io, key, step):
        """Capture fwd/bwd + update of this bucket into one CUDA graph."""
        g = torch.cuda.CUDAGraph()
        with _no_gc():
            with torch.cuda.graph(g, stream=_lib.context().compute_stream, **self._capture_kw()):
                out3, sink = self._fwd_bwd(io, key, step)
                self._update(out3, sink)
        self._graphs[key] = g
        torch.cuda.synchronize()

    def refresh_seeds(self, step: int):
        """Write this step's per-site dropout seeds (and the next step's, for the
        mask bank) into the pinned staging buffers."""
        t = self.cfg.train
        seeds = self.model.seed_table(self.device)
        self.model.register_seeds(seeds, t.seed, step, t.p_drop)
        seeds.write_host()
        if self.masks is not None and self._early_masks and t.p_drop > 0.0:
            self._stage_next_seeds(step)

    def _prestage(self, step: int):
        """Host work of `step` done ahead, while the device runs the previous step:
        build + validate the batch and stage it and the site seeds into the pinned
        buffers (the previous step's copies out of them have completed)."""
        try:
            batch = self.task.batch(step)
            validate_batch(batch, self.cfg.model)
        except Exception as exc:                       # raised by that step's call
            self._pre = (step, None, None, exc)
            return
        b, l = np.asarray(batch.src).shape
        key = ("train", b, l)
        if key not in self._graphs:
            self._pre = None
            return
        self._io_for(b, l).stage(batch)
        self.refresh_seeds(step)
        self._pre = (step, batch, key, None)

    def train_step(self, step: int, trace=None) -> StepMetrics:
        t0 = time.perf_counter()
        pre, self._pre = self._pre, None
        if pre is not None and pre[0] == step:
            if pre[3] is not None:
                raise pre[3]
            batch, key, staged = pre[1], pre[2], True
        else:
            batch = self.task.batch(step)
            validate_batch(batch, self.cfg.model)
            key, staged = ("train",) + tuple(np.asarray(batch.src).shape), False
        b, l = key[1], key[2]
        if self.arena is None or not self.arena.has_plan(key):
            raise DataError(f"no arena plan for batch shape {key}; call setup_arena()")
        io = self._io_for(b, l)
        graphed = self.use_graphs and key in self._graphs
        if graphed:
            if not staged:
                io.stage(batch)
                self.refresh_seeds(step)
            self._graphs[key].replay()
            if self._overlap_host:
                self._consumed.synchronize()           # inputs are on the device
                self._prestage(step + 1)
        else:
            io.stage(batch)
            self._run(io, key, step, graphed=False)
        if graphed:
            # the metrics copy (issued before the optimizer) has landed; the update
            # and the next step's mask draw may still run, and everything enqueued
            # after this call is stream-ordered behind them
            self._metrics_ev.synchronize()
        else:
            torch.cuda.current_stream().synchronize()
        loss, count, correct, applied, nonfinite = self._host_out.tolist()
        if self.use_graphs and key not in self._graphs:
            self._capture(io, key, step + 1)
        applied = bool(applied)
        skipped = not applied
        if applied:
            self.applied_steps += 1
        else:
            self.skip_count += 1
        dt = time.perf_counter() - t0
        count = int(count)
        return StepMetrics(step=step, loss=loss / max(count, 1), tokens=count,
                           accuracy=correct / max(count, 1),
                           tokens_per_sec=count / dt if dt > 0 else 0.0,
                           arena_high_water=self.arena.high_water, skipped=skipped,
                           nonfinite=int(nonfinite) if np.isfinite(loss) else 0)

    def evaluate(self, n_batches: int = 8) -> float:
        """Teacher-forced next-token accuracy on fresh batches, dropout off."""
        correct = total = 0
        for i in range(n_batches):
            batch = self.task.batch(EVAL_STEP_BASE + i)
            key = ("eval",) + tuple(np.asarray(batch.src).shape)
            self.arena.begin(key)
            out = self.model.forward_backward(self.pviews, batch, p_drop=0.0,
                                              alpha=self.cfg.train.alpha, seed=self.cfg.train.seed,
                                              step=EVAL_STEP_BASE + i, arena=self.arena,
                                              compute_grads=False)
            self.arena.end()
            correct += out.correct
            total += out.token_count
        return correct / max(total, 1)

    # -- checkpointing (F/engine.py:189-208, F/checkpoint.py) ----------------------------

    def checkpoint_tensors(self):
        torch.cuda.synchronize()
        tensors = [("params16", self.ws.params16.cpu().numpy()),
                   ("moments_m", self.ws.m32.cpu().numpy())]
        if self.ws.v32 is not None:
            tensors.append(("moments_v", self.ws.v32.cpu().numpy()))
        tensors.append(("applied_steps", np.array([self.applied_steps], dtype=np.float32)))
        return tensors

    def save(self, path: str, step: int) -> None:
        ckpt.save_checkpoint(path, step, self.checkpoint_tensors())

    def restore(self, path: str) -> int:
        step, tensors = ckpt.load_checkpoint(path)
        if tensors["params16"].size != self.ws.n_elements:
            raise DataError("checkpoint parameter count does not match the model")
        self.ws.params16.copy_(torch.from_numpy(tensors["params16"]).to(self.device))
        self.ws.m32.copy_(torch.from_numpy(tensors["moments_m"]).to(self.device))
        if self.ws.v32 is not None:
            self.ws.v32.copy_(torch.from_numpy(tensors["moments_v"]).to(self.device))
        self.applied_steps = int(tensors["applied_steps"][0])
        self._applied_dev.fill_(self.applied_steps)
        return step
