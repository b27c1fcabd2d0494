"""Pre-LayerNorm encoder/decoder built from the libls2 fused kernels.

Drop-in for F/model.py (same names, signatures, stash/LIFO discipline, packed
cross-attention and the "encoder gradient only after decoder layer 0"
ordering contract).  B200-specific choices, all invisible at the API:

* activations are stored in the parameters' dtype (fp16 on the training
  path; f32/f64 reproduce the reference's compute dtypes for parity tests);
* the attention contractions read Q/K/V straight out of the fused [B,L,3d]
  projection and write the context straight into [B,L,d] (two-level
  pointer-array cuBLAS batches), so there are no head split/merge copies;
* 1/sqrt(hd) is folded into the QK^T GEMM alpha and the softmax backward;
* dropout and relu masks are 1-bit device masks;
* parameter gradients are written directly into the fp32 gradient workspace
  (GEMM output / column-sum / LayerNorm partial reductions), never staged;
* per-step dropout seeds live in a small device table filled by one H2D copy,
  so a captured CUDA graph of the whole step replays with fresh masks.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import attention as ATT
from . import gradients as G
from . import kernels as K
from .errors import ConfigError, IncompleteGradientSet, SequenceTooLong, ShapeMismatch, TokenOutOfRange
from .kernels import AttentionMask, DropoutMask, EmbeddingConfig, LNCache, ReluMask, SoftmaxCache
from .memplan import NullArena
from .numerics import derive_seed, rand_uniform_array


# ---------------------------------------------------------------------------
# configuration and parameters (F/model.py:30-127)
# ---------------------------------------------------------------------------

@dataclass
class ModelConfig:
    n_enc: int = 2
    n_dec: int = 2
    d_model: int = 32
    n_heads: int = 4
    d_ff: int = 128
    vocab: int = 32
    max_len: int = 16
    pre_ln: bool = True
    tie_embeddings: bool = True
    learned_positional: bool = True
    eps: float = 1e-5
    embed_scale: float | None = None
    # "transformer": the reference's encoder-decoder; "encoder": a BERT-shaped
    # encoder with a tied masked-LM criterion (BASELINE.json configs[3])
    arch: str = "transformer"

    def __post_init__(self):
        if self.arch not in ("transformer", "encoder"):
            raise ConfigError(f"unknown arch {self.arch!r}")
        if self.d_model % self.n_heads:
            raise ConfigError(f"d_model {self.d_model} not divisible by n_heads {self.n_heads}")
        if self.vocab < 2:
            raise ConfigError("vocab must be >= 2")
        if not self.pre_ln:
            raise ConfigError("only the pre-LayerNorm layout is implemented")

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads

    @property
    def scale(self) -> float:
        return self.embed_scale if self.embed_scale is not None else math.sqrt(self.d_model)


def _layer_spec(pre: str, d: int, dff: int, decoder: bool):
    s = [(pre + "ln1.w", (d,)), (pre + "ln1.b", (d,)), (pre + "attn.wqkv", (3 * d, d)),
         (pre + "attn.bqkv", (3 * d,)), (pre + "attn.wo", (d, d)), (pre + "attn.bo", (d,)),
         (pre + "ln2.w", (d,)), (pre + "ln2.b", (d,))]
    if decoder:
        s += [(pre + "cross.wq", (d, d)), (pre + "cross.bq", (d,)), (pre + "cross.wo", (d, d)),
              (pre + "cross.bo", (d,)), (pre + "ln3.w", (d,)), (pre + "ln3.b", (d,))]
    return s + [(pre + "ffn.w1", (dff, d)), (pre + "ffn.b1", (dff,)), (pre + "ffn.w2", (d, dff)),
                (pre + "ffn.b2", (d,))]


def param_spec(cfg: ModelConfig):
    """(name, shape) list; the order defines the workspace layout (F/model.py:82-97)."""
    d, dff = cfg.d_model, cfg.d_ff
    spec = [("tok_emb", (cfg.vocab, d))]
    if cfg.learned_positional:
        spec.append(("pos_emb", (cfg.max_len, d)))
    for i in range(cfg.n_enc):
        spec += _layer_spec(f"enc{i}.", d, dff, False)
    if cfg.arch == "encoder":
        return spec + [("enc_ln.w", (d,)), ("enc_ln.b", (d,))]
    spec += [("enc_ln.w", (d,)), ("enc_ln.b", (d,)),
             ("cross_kv.w", (2 * cfg.n_dec * d, d)), ("cross_kv.b", (2 * cfg.n_dec * d,))]
    for i in range(cfg.n_dec):
        spec += _layer_spec(f"dec{i}.", d, dff, True)
    spec += [("dec_ln.w", (d,)), ("dec_ln.b", (d,))]
    if not cfg.tie_embeddings:
        spec.append(("out_proj.w", (cfg.vocab, d)))
    return spec


def init_params(cfg: ModelConfig, seed: int, device=None) -> dict:
    """Counter-RNG init on the device, bit-identical to F/model.py:100-118."""
    ctx = _lib.context(device)
    params = {}
    for idx, (name, shape) in enumerate(param_spec(cfg)):
        n = int(np.prod(shape))
        leaf = name.rsplit(".", 1)[-1]
        if leaf == "w" and "ln" in name:
            params[name] = torch.ones(shape, dtype=torch.float32, device=ctx.device)
        elif leaf in ("b", "bqkv", "bo", "bq", "b1", "b2"):
            params[name] = torch.zeros(shape, dtype=torch.float32, device=ctx.device)
        else:
            u = rand_uniform_array(derive_seed(seed, idx), 0, n, device=ctx.device)
            if "emb" in name or name == "out_proj.w":
                lim = 0.02 * math.sqrt(3.0)
            else:
                fo, fi = (shape[0], shape[1]) if len(shape) == 2 else (shape[0], shape[0])
                lim = math.sqrt(6.0 / (fi + fo))
            params[name] = ((2.0 * u - 1.0) * lim).to(torch.float32).reshape(shape)
    return params


def sinusoidal_table(max_len: int, d: int, dtype=torch.float32, device=None) -> torch.Tensor:
    """Fixed positional table (F/model.py:121-127), built in float64 then cast."""
    pos = np.arange(max_len, dtype=np.float64)[:, None]
    j = np.arange(d, dtype=np.float64)[None, :]
    ang = pos / np.power(10000.0, 2.0 * np.floor(j / 2.0) / d)
    tab = np.where(j % 2 == 0, np.sin(ang), np.cos(ang))
    return torch.from_numpy(tab).to(device or _lib.context().device).to(dtype)


# ---------------------------------------------------------------------------
# layer weight views (F/model.py:134-172)
# ---------------------------------------------------------------------------

_ENC_FIELDS = [("ln1_w", "ln1.w"), ("ln1_b", "ln1.b"), ("wqkv", "attn.wqkv"), ("bqkv", "attn.bqkv"),
               ("wo", "attn.wo"), ("bo", "attn.bo"), ("ln2_w", "ln2.w"), ("ln2_b", "ln2.b"),
               ("w1", "ffn.w1"), ("b1", "ffn.b1"), ("w2", "ffn.w2"), ("b2", "ffn.b2")]
_DEC_EXTRA = [("cross_wq", "cross.wq"), ("cross_bq", "cross.bq"), ("cross_wo", "cross.wo"),
              ("cross_bo", "cross.bo"), ("ln3_w", "ln3.w"), ("ln3_b", "ln3.b")]


class EncoderLayerWeights:
    _fields = _ENC_FIELDS

    def __init__(self, **kw):
        for k, v in kw.items():
            setattr(self, k, v)

    @classmethod
    def from_params(cls, params, prefix: str):
        return cls(**{attr: params[prefix + key] for attr, key in cls._fields})


class DecoderLayerWeights(EncoderLayerWeights):
    _fields = _ENC_FIELDS + _DEC_EXTRA


# ---------------------------------------------------------------------------
# packed cross-attention K/V projection (F/model.py:179-260)
# ---------------------------------------------------------------------------

@dataclass
class PackedCrossWeights:
    """[Wkey_0; ..; Wkey_{n-1}; Wval_0; ..; Wval_{n-1}]  ([2*n*d, d])."""

    w: torch.Tensor
    b: torch.Tensor
    n_layers: int
    d: int

    def key_slice(self, i: int):
        return self.w[i * self.d:(i + 1) * self.d]

    def value_slice(self, i: int):
        return self.w[(self.n_layers + i) * self.d:(self.n_layers + i + 1) * self.d]


def pack_cross_weights(keys, values, key_biases, value_biases) -> PackedCrossWeights:
    n = len(keys)
    if n < 1 or len(values) != n or len(key_biases) != n or len(value_biases) != n:
        raise ShapeMismatch("need matching, non-empty key/value weight lists")
    ks = [K.dev(m) for m in keys]
    vs = [K.dev(m) for m in values]
    d = ks[0].shape[1]
    for m in ks + vs:
        if tuple(m.shape) != (d, d):
            raise ShapeMismatch(f"cross projection must be [{d}x{d}], got {tuple(m.shape)}")
    w = torch.cat(ks + vs, dim=0)
    b = torch.cat([K.dev(v).reshape(-1) for v in list(key_biases) + list(value_biases)])
    return PackedCrossWeights(w=w, b=b, n_layers=n, d=d)


def unpack_cross_weights(pw: PackedCrossWeights):
    n, d = pw.n_layers, pw.d
    keys = [pw.key_slice(i).clone() for i in range(n)]
    values = [pw.value_slice(i).clone() for i in range(n)]
    kb = [pw.b[i * d:(i + 1) * d].clone() for i in range(n)]
    vb = [pw.b[(n + i) * d:(n + i + 1) * d].clone() for i in range(n)]
    return keys, values, kb, vb


def _as_dt(t, dt):
    t = t if isinstance(t, torch.Tensor) else K.dev(t)
    return t if t.dtype == dt else t.to(dt)


def _linear(x2d, w, b, out2d):
    """out = x @ w^T (+ b): one cuBLASLt GEMM with the bias fused as its epilogue
    (fallback: cuBLAS GEMM + libls2 bias-add where Lt has no algorithm)."""
    dt = out2d.dtype
    wt = _as_dt(w, dt)
    bb = None if b is None else _as_dt(b, dt).contiguous()
    ctx = _lib.context()
    if dt != torch.float64 and x2d.is_contiguous() and wt.is_contiguous() and out2d.is_contiguous() \
            and x2d.dtype == dt:
        m, k = x2d.shape
        n = wt.shape[0]
        key = (m, n, k, dt, bb is not None)
        if key not in ctx.lt_unsupported:
            try:
                _lib.call("ls2_gemm_lt", ctx.blas_handle(), 0, 1, m, n, k, 1.0, x2d.data_ptr(), k,
                          wt.data_ptr(), k, 0.0, out2d.data_ptr(), n, _lib.ptr(bb),
                          _lib.dtype_code(dt), _lib.dtype_code(dt), _lib.stream_handle())
                return out2d
            except Exception:
                ctx.lt_unsupported.add(key)
    K.gemm(x2d, wt, trans_b=True, out=out2d)
    if bb is not None:
        _lib.call("ls2_bias_add", out2d.data_ptr(), bb.data_ptr(), out2d.shape[0],
                  out2d.shape[1], _lib.dtype_code(out2d), _lib.stream_handle())
    return out2d


def packed_kv_forward(enc_out, pw: PackedCrossWeights, arena=None):
    """One GEMM of enc_out against the packed weights, then a 2n-way view split."""
    arena = arena or NullArena()
    enc_out = enc_out if isinstance(enc_out, torch.Tensor) else K.dev(enc_out)
    if enc_out.shape[-1] != pw.d:
        raise ShapeMismatch(f"enc_out feature dim {enc_out.shape[-1]} != {pw.d}")
    b, ls, d = enc_out.shape
    n = pw.n_layers
    if enc_out.dtype in (torch.float16, torch.bfloat16):
        dt = enc_out.dtype                       # storage dtype of the training path
    else:
        dt = K.compute_dtype(enc_out, pw.w)      # reference dtype rule
    buf = arena.alloc((b, ls, 2 * n * d), dt)
    _linear(_as_dt(enc_out, dt).reshape(b * ls, d), pw.w, pw.b, buf.view(b * ls, 2 * n * d))
    pairs = [(buf[..., i * d:(i + 1) * d], buf[..., (n + i) * d:(n + i + 1) * d]) for i in range(n)]
    return pairs, buf


def packed_kv_backward(dks, dvs, enc_out, pw: PackedCrossWeights, arena=None, packed=None,
                       sink=None, bias_done: bool = False):
    """dx = sum_i Wkey_i^T dK_i + Wval_i^T dV_i via one packed GEMM; (dx, dw, db).

    Raises IncompleteGradientSet unless every decoder layer contributed.  When
    the dK_i/dV_i are already views of one packed buffer (`packed`), no copy is
    made.  With a sink the weight/bias grads go straight into it (dw, db None)."""
    arena = arena or NullArena()
    n = pw.n_layers
    if len(dks) != n or len(dvs) != n or any(g is None for g in dks) or any(g is None for g in dvs):
        raise IncompleteGradientSet("missing dK/dV contribution for some decoder layer")
    enc_out = enc_out if isinstance(enc_out, torch.Tensor) else K.dev(enc_out)
    b, ls, d = enc_out.shape
    dt = dks[0].dtype if isinstance(dks[0], torch.Tensor) else K.compute_dtype(enc_out, dks[0])
    own = packed is None
    if own:
        dy = arena.alloc((b, ls, 2 * n * d), dt)
        for i in range(n):
            dy[..., i * d:(i + 1) * d].copy_(K.dev(dks[i]).view(b, ls, d))
            dy[..., (n + i) * d:(n + i + 1) * d].copy_(K.dev(dvs[i]).view(b, ls, d))
    else:
        dy = packed
    dy2 = dy.view(b * ls, 2 * n * d)
    dx = arena.alloc((b, ls, d), dt)
    K.gemm(dy2, _as_dt(pw.w, dt), out=dx.view(b * ls, d))
    e2 = _as_dt(enc_out, dt).reshape(b * ls, d)
    dw = db = None
    if sink is not None:
        _wgrad(sink, "cross_kv.w", dy2, e2)
        if not bias_done:          # else: left by the attention backward kernels
            _colsum_grad(sink, "cross_kv.b", dy2)
    else:
        dw = K.gemm(dy2, e2, trans_a=True)
        db = G.column_sum(dy2)
    if own:
        arena.free(dy)
    return dx, dw, db


# ---------------------------------------------------------------------------
# activation stash and gradient sinks (F/model.py:267-311)
# ---------------------------------------------------------------------------

class ActivationStash:
    """LIFO store of saved activations; every entry is consumed exactly once."""

    def __init__(self):
        self._items: list = []

    def push(self, tag: str, value):
        self._items.append((tag, value))

    def pop(self, tag: str):
        if not self._items:
            raise ShapeMismatch(f"stash empty, wanted {tag!r}")
        got, value = self._items.pop()
        if got != tag:
            raise ShapeMismatch(f"stash order broken: wanted {tag!r}, top is {got!r}")
        return value

    def drain(self, arena):
        while self._items:
            _, value = self._items.pop()
            if isinstance(value, torch.Tensor):
                arena.free(value)

    def __len__(self):
        return len(self._items)


class GradSink:
    """Accumulates named parameter gradients (dict-backed by default)."""

    def __init__(self, store: dict | None = None):
        self.store = store if store is not None else {}

    def add(self, name: str, value):
        if name in self.store:
            self.store[name] += value
        else:
            self.store[name] = value.clone()

    def target(self, name: str):
        """(view, beta) to write a gradient in place, or None to use add()."""
        return None


class _ViewSink(GradSink):
    """Writes into preallocated views of the fp32 gradient workspace; the first
    producer of a name overwrites (beta=0), later producers accumulate."""

    def __init__(self, store: dict, defer: bool = False, lane: bool = False,
                 wgrad_group: int | None = None):
        super().__init__(store)
        self.use_lane = bool(lane)
        # weight-gradient GEMMs batched across layers (_WgradBatch): flushed every
        # `wgrad_group` layers (0: only at the end of backward); None: off
        self.wgrad_group = wgrad_group
        self.written: set = set()
        # deferred column sums: the producer leaves per-block partials in an arena
        # buffer and the engine finishes them all inside the fp16 narrow pass
        self.defer_enabled = defer
        self.deferred: list = []          # (name, buf, nblk, stride, k, cols)
        self.arena = None
        self.lane = None                  # _Lane for weight-gradient GEMMs (engine path)
        self.on_ready = None              # engine hook: gradients of these names are final
        self.on_layer_done = None         # engine hook: raw ready() prefixes
        self.totals = None                # (loss, count, correct) once the criterion ran

    def ready(self, prefixes):
        """Backward has finished every parameter whose name starts with one of
        `prefixes` (None: all remaining) — the data-parallel exchange may start,
        and that layer's dropout bits are dead (mask bank)."""
        if self.on_layer_done is not None:
            self.on_layer_done(prefixes)
        if self.on_ready is not None:
            names = None if prefixes is None else \
                [n for n in self.store if any(n.startswith(p) for p in prefixes)]
            self.on_ready(names)

    def _settle(self, name: str):
        """A second producer of `name` writes now: issue its pending batched GEMM."""
        lane = self.lane
        if lane is not None and name in getattr(lane, "pending", ()):
            lane.flush()

    def add(self, name: str, value):
        self._settle(name)
        if name in self.written:
            self.store[name] += value
        else:
            self.store[name].copy_(value)
            self.written.add(name)

    def target(self, name: str):
        self._settle(name)
        beta = 1 if name in self.written else 0
        self.written.add(name)
        return self.store[name], beta

    def defer_buffer(self, names, nblk: int, np_: int, cols: int):
        """Arena buffer for nblk x np_ x cols partials of `names`, or None."""
        for n in names:
            self._settle(n)
        if not self.defer_enabled or self.arena is None or nblk <= 0 or \
                any(n in self.written for n in names):
            return None
        buf = self.arena.alloc((nblk * np_ * cols,), torch.float64)
        for k, n in enumerate(names):
            self.written.add(n)
            self.deferred.append((n, buf, nblk, np_ * cols, k, cols))
        return buf

    def deferred_buffers(self):
        seen, out = set(), []
        for _, buf, *_ in self.deferred:
            if id(buf) not in seen:
                seen.add(id(buf))
                out.append(buf)
        return out


class _Lane:
    """Side-stream lane for weight-gradient GEMMs (off the critical path).

    dW = dy^T x is only consumed by the optimizer, so it runs on a low-priority
    stream with its own cuBLAS workspace while the main stream continues with
    the data-gradient chain.  Arena buffers such a GEMM reads are held: their
    frees are deferred to the next join(), where the main stream first waits for
    the lane.  The same alloc/free sequence happens in the arena's dry run, so
    the planned lifetimes include the hold."""

    def __init__(self, arena):
        ctx = _lib.context()
        self.main = torch.cuda.current_stream()
        self.side = ctx.side_stream
        self.arena = arena
        self.held: set = set()
        self.deferred: list = []
        self.pending = False

    def wgrad(self, name, dy2d, x2d, out2d, beta):
        self.run(lambda: K.gemm(dy2d, x2d, trans_a=True, out=out2d, beta=float(beta)), dy2d, x2d)

    def postpone(self, prefixes) -> bool:
        return False

    def run(self, fn, *reads):
        ev = torch.cuda.Event()
        ev.record(self.main)
        self.side.wait_event(ev)
        with torch.cuda.stream(self.side):
            fn()
        for t in reads:
            self.held.add(t.data_ptr())
        self.pending = True

    def free(self, t):
        if t.data_ptr() in self.held:
            self.deferred.append(t)
        else:
            self.arena.free(t)

    def join(self):
        if self.pending:
            ev = torch.cuda.Event()
            ev.record(self.side)
            self.main.wait_event(ev)
            self.pending = False
        self.held.clear()
        for t in self.deferred:
            self.arena.free(t)
        self.deferred.clear()

    flush = join


class _WgradBatch:
    """Weight-gradient GEMMs batched across layers (engine path).

    dW = dy^T x is consumed only by the optimizer (or by the data-parallel
    exchange of its bucket), so `_wgrad` enqueues it here and `flush()` issues
    every pending product of one shape as ONE cuBLAS pointer-array batch
    (K.gemm_list): the Transformer-base step's 24 [512 x 512] x 4096 weight
    gradients take ~55 us as one batch against ~215 us one by one, the FFN ones
    84 vs 153 us per 12 (profiles/r3a_wgrad_batch.jsonl).  The engine flushes
    every `group` layers (0: once, at the end of backward).  Like the lane, the
    arena buffers a pending GEMM reads are held (their frees wait for the
    flush, in the planner's dry run too), and the readiness of the layers whose
    gradients are pending (`_ready`: the DP exchange of their buckets) is
    postponed to the flush.  Products with large outputs (the vocabulary
    projection) gain nothing from batching and run at once."""

    MAX_OUT = 1 << 22          # outputs of more elements run immediately

    def __init__(self, arena, group: int):
        self.arena, self.group = arena, int(group)
        self.items: list = []          # (name, dy2d, x2d, out2d, beta)
        self.pending: set = set()
        self.held: set = set()
        self.deferred: list = []
        self.ready_q: list = []
        self.sink = None
        self.layers = 0

    def wgrad(self, name, dy2d, x2d, out2d, beta):
        if out2d.numel() > self.MAX_OUT or not all(t.is_contiguous() for t in (dy2d, x2d, out2d)):
            K.gemm(dy2d, x2d, trans_a=True, out=out2d, beta=float(beta))
            return
        self.items.append((name, dy2d, x2d, out2d, float(beta)))
        self.pending.add(name)
        self.held.add(dy2d.data_ptr())
        self.held.add(x2d.data_ptr())

    def free(self, t):
        if t.data_ptr() in self.held:
            self.deferred.append(t)
        else:
            self.arena.free(t)

    def postpone(self, prefixes) -> bool:
        if not self.items:
            return False
        self.ready_q.append(prefixes)
        return True

    def join(self):
        self.layers += 1
        if self.group > 0 and self.layers >= self.group:
            self.flush()

    def flush(self):
        groups: dict = {}
        for name, dy, x, out, beta in self.items:
            key = (tuple(dy.shape), tuple(x.shape), dy.dtype, out.dtype, beta)
            groups.setdefault(key, []).append((dy, x, out))
        for (_, _, _, _, beta), its in groups.items():
            K.gemm_list([i[0] for i in its], [i[1] for i in its], [i[2] for i in its],
                        trans_a=True, beta=beta)
        self.items.clear()
        self.pending.clear()
        self.layers = 0
        self.held.clear()
        for t in self.deferred:
            self.arena.free(t)
        self.deferred.clear()
        q, self.ready_q = self.ready_q, []
        for prefixes in q:
            _ready_now(self.sink, prefixes)


def _open_lane(sink, arena, dt):
    """(lane, arena facade, join) for the backward pass: the side-stream lane
    (LS2_WGRAD_LANE=1), the cross-layer weight-gradient batch, or neither."""
    if dt == torch.float64:
        return None, arena, (lambda: None)
    if getattr(sink, "use_lane", False):
        lane = _Lane(arena)
    elif getattr(sink, "wgrad_group", None) is not None:
        lane = _WgradBatch(arena, sink.wgrad_group)
        lane.sink = sink
    else:
        return None, arena, (lambda: None)
    sink.lane = lane
    return lane, _LaneArena(arena, lane), lane.join


def _close_lane(sink, lane):
    if lane is not None:
        lane.flush()
        sink.lane = None


class _LaneArena:
    """Arena facade whose frees respect the lane's holds."""

    def __init__(self, arena, lane: _Lane):
        self._arena, self._lane = arena, lane

    def alloc(self, shape, dtype):
        return self._arena.alloc(shape, dtype)

    def free(self, t):
        self._lane.free(t)

    def __getattr__(self, name):
        return getattr(self._arena, name)


def _ready(sink, *prefixes):
    pre = list(prefixes) if prefixes != (None,) else None
    lane = getattr(sink, "lane", None)
    if lane is not None and lane.postpone(pre):
        return                       # its weight gradients are still pending
    _ready_now(sink, pre)


def _ready_now(sink, prefixes):
    fn = getattr(sink, "ready", None)
    if fn is not None:
        fn(prefixes)


def _defer(sink, names, nblk, np_, cols):
    fn = getattr(sink, "defer_buffer", None)
    return fn(names, nblk, np_, cols) if fn is not None else None


def _aligned(*ts) -> bool:
    return all(t is None or (t.is_contiguous() and t.data_ptr() % 16 == 0) for t in ts)


def _colsum_nblk(rows, cols, t) -> int:
    if t.dtype == torch.float64:
        return 0
    return int(_lib._lib.ls2_colsum_nblk(rows, cols, _lib.dtype_code(t)))


def _wgrad(sink, name, dy2d, x2d):
    """dW = dy^T x straight into the sink (cuBLAS, fp32 output); through the
    sink's lane (side stream or cross-layer batch) when it has one."""
    tgt = sink.target(name)
    if tgt is None:
        sink.add(name, K.gemm(dy2d, x2d, trans_a=True))
        return
    v, beta = tgt
    out2d = v.view(dy2d.shape[1], x2d.shape[1])
    lane = getattr(sink, "lane", None)
    if lane is not None:
        lane.wgrad(name, dy2d, x2d, out2d, beta)
    else:
        K.gemm(dy2d, x2d, trans_a=True, out=out2d, beta=float(beta))


def _colsum_grad(sink, name, x2d):
    rows, cols = x2d.shape
    if _aligned(x2d):
        buf = _defer(sink, [name], _colsum_nblk(rows, cols, x2d), 1, cols)
        if buf is not None:
            G.column_sum(x2d, partials_out=buf)
            return
    tgt = sink.target(name)
    if tgt is None:
        sink.add(name, G.column_sum(x2d))
    else:
        v, beta = tgt
        G.column_sum(x2d, out=v, beta=beta)


def _bias_target(sink, name):
    tgt = sink.target(name)
    return (None, 0, False) if tgt is None else (tgt[0], tgt[1], True)


def _ln_targets(sink, pp, ln):
    tw, tb = sink.target(pp + ln + ".w"), sink.target(pp + ln + ".b")
    if tw is None or tb is None or tw[1] != tb[1]:
        return None, None, 0
    return tw[0], tb[0], tw[1]


def _ln_bwd(sink, pp, ln, du, x_in, w, mu, sg, out, dres):
    wt = _as_dt(w, du.dtype)
    rows, cols = du.numel() // du.shape[-1], du.shape[-1]
    if du.dtype != torch.float64 and _aligned(du, x_in, wt, out, dres):
        nblk = int(_lib._lib.ls2_layernorm_bwd_nblk(rows, cols))
        buf = _defer(sink, [pp + ln + ".w", pp + ln + ".b"], nblk, 2, cols)
        if buf is not None:
            G.layernorm_backward(du, x_in, wt, LNCache(mu, sg), out=out, dres=dres,
                                 partials_out=buf)
            return
    dwv, dbv, beta = _ln_targets(sink, pp, ln)
    _, dw, db = G.layernorm_backward(du, x_in, wt, LNCache(mu, sg), out=out,
                                     dres=dres, dw_out=dwv, db_out=dbv, beta=beta)
    if dwv is None:
        sink.add(pp + ln + ".w", dw)
        sink.add(pp + ln + ".b", db)


def _bdr_bwd(sink, name, dy, keep_bits, p_drop, out):
    mask = DropoutMask(p=p_drop, bits=keep_bits, shape=tuple(dy.shape))
    rows, cols = dy.numel() // dy.shape[-1], dy.shape[-1]
    if _aligned(dy, out):
        buf = _defer(sink, [name], _colsum_nblk(rows, cols, dy), 1, cols)
        if buf is not None:
            G.bias_dropout_residual_backward(dy, mask, out=out, partials_out=buf)
            return
    dv, beta, direct = _bias_target(sink, name)
    _, db, _ = G.bias_dropout_residual_backward(dy, mask, out=out, dbias_out=dv, beta=beta)
    if not direct:
        sink.add(name, db)


def _brd_bwd(sink, name, dz, keep_bits, relu_bits, p_drop, out):
    mask = DropoutMask(p=p_drop, bits=keep_bits, shape=tuple(dz.shape))
    relu = ReluMask(bits=relu_bits, shape=tuple(dz.shape))
    rows, cols = dz.numel() // dz.shape[-1], dz.shape[-1]
    if _aligned(dz, out):
        buf = _defer(sink, [name], _colsum_nblk(rows, cols, dz), 1, cols)
        if buf is not None:
            G.bias_relu_dropout_backward(dz, mask, relu, out=out, partials_out=buf)
            return
    dv, beta, direct = _bias_target(sink, name)
    _, db = G.bias_relu_dropout_backward(dz, mask, relu, out=out, dbias_out=dv, beta=beta)
    if not direct:
        sink.add(name, db)


# ---------------------------------------------------------------------------
# attention helpers (F/model.py:318-328) — views, never copies
# ---------------------------------------------------------------------------

def _heads(x, n_heads: int):
    """[B, L, d] -> [B, N, L, d/N] strided view."""
    b, l, d = x.shape
    return x.view(b, l, n_heads, d // n_heads).transpose(1, 2) if x.is_contiguous() else \
        x.unflatten(-1, (n_heads, d // n_heads)).transpose(1, 2)


def _merge_heads(xh, out):
    """[B, N, L, hd] -> [B, L, d] copy into out (API helper; the model writes
    attention contexts directly in merged layout)."""
    b, n, l, hd = xh.shape
    out.view(b, l, n, hd).copy_(xh.transpose(1, 2))
    return out


def _qkv_heads(qkv, n_heads: int):
    d = qkv.shape[-1] // 3
    return tuple(_heads(qkv[..., i * d:(i + 1) * d], n_heads) for i in range(3))


class SeedTable:
    """Per-step dropout seeds on the device (one H2D copy per step).

    slot(group_base, site, k) -> 1-element uint64 CUDA view holding
    derive_seed(group_base, site, k); kernels read it through seed_ptr."""

    def __init__(self, device, capacity: int = 256):
        self.host = torch.zeros(capacity, dtype=torch.int64).pin_memory()
        self.dev = torch.zeros(capacity, dtype=torch.int64, device=device)
        self.index: dict = {}
        self.values: list = []
        self._evt = None

    def reset(self):
        self.index.clear()
        self.values.clear()

    def set_step(self, step: int):
        """Slot 0 holds the step number (the mask bank's stamp compares with it)."""
        self.slot_value("__step__", step)

    def step_slot(self):
        return self.slot_value("__step__", None)

    def slot_value(self, name: str, value):
        key = (name,)
        i = self.index.get(key)
        if i is None:
            i = self.index[key] = len(self.values)
            self.values.append(0 if value is None else value)
        elif value is not None:
            self.values[i] = value
        return self.dev[i:i + 1]

    def slot(self, base: int, *tags: int):
        key = (base,) + tags
        i = self.index.get(key)
        if i is None:
            i = self.index[key] = len(self.values)
            self.values.append(derive_seed(base, *tags) if tags else base)
        return self.dev[i:i + 1]

    def upload(self):
        span = self.stage_span()
        self.dev[:len(self.values)].copy_(self.host[:len(self.values)], non_blocking=True)
        self.uploaded()
        return span

    def stage_span(self):
        """Fill the pinned staging buffer; (dst, src, nbytes) of the H2D copy the
        caller issues (engine: one ls2_copy_spans launch for every step input)."""
        n = len(self.values)
        if n > self.host.numel():
            raise ShapeMismatch("seed table overflow")
        self.write_host(sync=not torch.cuda.is_current_stream_capturing())
        return (self.dev.data_ptr(), self.host.data_ptr(), 8 * n)

    def uploaded(self):
        """After the copy is enqueued: the next write_host waits for it (eager)."""
        if not torch.cuda.is_current_stream_capturing():
            self._evt = torch.cuda.Event()
            self._evt.record()

    def write_host(self, sync: bool = True):
        """Fill the pinned staging buffer (waits until the previous copy ran)."""
        if sync and self._evt is not None:
            self._evt.synchronize()
        n = len(self.values)
        vals = np.array([v - (1 << 64) if v >= (1 << 63) else v for v in self.values], dtype=np.int64)
        self.host[:n].copy_(torch.from_numpy(vals))


class _LayerSeed:
    """Seed handle handed to a layer: int (reference API) or table-backed."""

    def __init__(self, table: SeedTable, base: int):
        self.table, self.base = table, base

    def site(self, site: int, k: int):
        return self.table.slot(self.base, site, k)


def _site_seed(seed, site: int, k: int):
    if isinstance(seed, _LayerSeed):
        return seed.site(site, k)
    return derive_seed(seed, site, k)


class MaskBank:
    """Keep bits of every forward dropout site of a step, drawn by ONE launch.

    The reference draws each site's mask inside its op (F/kernels.py:155-166,
    splitmix64 per element).  Drawing all of a step's sites with one
    ALU-dense ls2_dropout_bits_multi launch turns the memory-bound fused
    forward kernels (bias+ReLU+dropout, bias+dropout+residual(+LayerNorm),
    embedding) into pure streams that read 1 bit per element; the bits are
    identical.  Keep bit i of a site depends only on (site seed, i), so each
    site owns a fixed region sized for the largest batch shape and any shape
    reads a prefix: one layout for every bucket.

    The draw runs at the start of the step.  Optionally (LS2_EARLY_MASKS=1) the
    engine draws step t+1's bits beside step t's Adam and stamps them with t+1;
    step t+1 then finds stamp == its step and its in-step draw exits at once
    (any other order — first step, a skipped step number — draws in-step).  Sites are keyed
    by their seed slot in the step's SeedTable; the backward pass reads the
    same bits again.  The buffer lives outside the activation arena.
    """

    def __init__(self, device):
        self.device = device
        self.buf = None
        self.desc = None
        self.nsites = 0
        self.words = 0
        self.sites: dict = {}
        self.max_tokens = None            # (src, tgt) tokens of the largest batch shape
        self.stamp = torch.full((1,), -1, dtype=torch.int64, device=device)
        self.thresh = 0
        self.active = False

    def configure(self, max_src_tokens: int, max_tgt_tokens: int):
        self.max_tokens = (int(max_src_tokens), int(max_tgt_tokens))

    def prepare(self, sites_fn, src_tokens: int, tgt_tokens: int, thresh: int):
        """Lay the sites out once (sites_fn(src_tokens, tgt_tokens) -> [(slot, n)])."""
        if self.max_tokens is None:
            self.max_tokens = (src_tokens, tgt_tokens)
        if src_tokens > self.max_tokens[0] or tgt_tokens > self.max_tokens[1]:
            raise ShapeMismatch("batch larger than the mask bank's configured maximum")
        if self.desc is None:
            rows, woff, offs, spans = [], 0, {}, {}
            for slot, n, grp in sites_fn(*self.max_tokens):
                rows.append([slot, n, woff, 0])
                offs[slot] = 4 * woff
                spans.setdefault(grp, []).append(len(rows) - 1)
                woff += ((n + 31) // 32 + 3) // 4 * 4        # 16-byte aligned sites
            self.desc = torch.tensor(rows, dtype=torch.int64, device=self.device)
            self.nsites, self.words, self.sites = len(rows), woff, offs
            self.buf = torch.zeros(4 * woff, dtype=torch.uint8, device=self.device)
            # per-layer groups (contiguous in the layout): drawn one by one as the
            # backward pass releases them (engine, LS2_EARLY_MASKS=1)
            self.groups = {}
            for grp, idx in spans.items():
                w0 = rows[idx[0]][2]
                w1 = rows[idx[-1]][2] + ((rows[idx[-1]][1] + 31) // 32 + 3) // 4 * 4
                sub = [[rows[i][0], rows[i][1], rows[i][2] - w0, 0] for i in idx]
                self.groups[grp] = (torch.tensor(sub, dtype=torch.int64, device=self.device),
                                    len(sub), w1 - w0, 4 * w0)
        self.thresh = thresh

    def generate_group(self, grp: str, seeds_dev: torch.Tensor):
        desc, ns, words, off = self.groups[grp]
        _lib.call("ls2_dropout_bits_multi", desc.data_ptr(), ns, words, self.buf.data_ptr() + off,
                  seeds_dev.data_ptr(), self.thresh, None, None, _lib.stream_handle())

    def generate(self, seeds_dev: torch.Tensor, stamp=None, want=None, ctas_per_sm: int = 0):
        """Draw every site with the seeds in seeds_dev (skipped on the device
        when *stamp == *want); ctas_per_sm > 0 caps the draw's residency so a
        concurrent kernel keeps the rest of every SM."""
        _lib.call("ls2_dropout_bits_multi_ex", self.desc.data_ptr(), self.nsites, self.words,
                  self.buf.data_ptr(), seeds_dev.data_ptr(), self.thresh, _lib.ptr(stamp),
                  _lib.ptr(want), int(ctas_per_sm), _lib.stream_handle())

    def bits(self, seed, n: int):
        """Bank view for the site whose seed is the table slot `seed`, else None."""
        if not self.active or not isinstance(seed, torch.Tensor):
            return None
        off = self.sites.get(seed.storage_offset())
        return None if off is None else self.buf[off:off + _nbits(n)]

    def owns(self, t) -> bool:
        if self.buf is None:
            return False
        p = t.data_ptr()
        return self.buf.data_ptr() <= p < self.buf.data_ptr() + self.buf.numel()


_MASKS: MaskBank | None = None       # the bank of the forward_backward in flight

# chain fusion across layer boundaries (LS2_CHAIN_FUSE=0: off): a layer's FFN
# tail (bias+dropout+residual) runs fused with the LayerNorm that consumes its
# output (the next layer's ln1, or the stack's final LN), forward and backward
CHAIN_FUSE = os.environ.get("LS2_CHAIN_FUSE", "1") != "0"


def _bank_bits(seed, n: int):
    return _MASKS.bits(seed, n) if _MASKS is not None else None


class _BankArena:
    """Arena facade: bank views are not arena blocks, their frees are no-ops."""

    def __init__(self, arena, bank: MaskBank):
        self._arena, self._bank = arena, bank

    def alloc(self, shape, dtype):
        return self._arena.alloc(shape, dtype)

    def free(self, t):
        if not self._bank.owns(t):
            self._arena.free(t)

    def __getattr__(self, name):
        return getattr(self._arena, name)


def _stat_dtype(dt):
    return torch.float64 if dt == torch.float64 else torch.float32


def _nbits(n: int) -> int:
    return (n + 7) // 8


# ---------------------------------------------------------------------------
# encoder layer (F/model.py:335-510)
# ---------------------------------------------------------------------------

def _fusable_rows(*ts) -> bool:
    """Row-fused kernels need 16-bit/f32 storage, d % 8 == 0, d <= 1024, 16-B alignment."""
    t0 = ts[0]
    if t0.dtype not in (torch.float16, torch.bfloat16, torch.float32):
        return False
    d = t0.shape[-1]
    if d % 8 or d > 1024:
        return False
    return all(t is None or (t.is_contiguous() and t.data_ptr() % 16 == 0) for t in ts)


def _tail_ln_core(proj, bias, res, p_drop, seed, ln_w, ln_b, eps, arena):
    """y = bias_dropout_residual(proj, bias, res) and u = LN(y) in one fused
    pass when possible (ls2_bdr_layernorm_fwd), else the two reference-shaped
    ops; returns (y, keep bits, mu, sigma, u)."""
    b, l, d = proj.shape
    r, dt = b * l, proj.dtype
    sdt = _stat_dtype(dt)
    y = arena.alloc((b, l, d), dt)
    banked = _bank_bits(seed, r * d) if p_drop > 0.0 else None
    keep = banked if banked is not None else arena.alloc((_nbits(r * d),), torch.uint8)
    mu, sg = arena.alloc((r,), sdt), arena.alloc((r,), sdt)
    u = arena.alloc((b, l, d), dt)
    bb, lw, lb = _as_dt(bias, dt), _as_dt(ln_w, dt), _as_dt(ln_b, dt)
    if _fusable_rows(proj, bb, res, y, lw, lb, u) and res.dtype == dt:
        use, thresh, ds = K._drop_args(p_drop)
        sv, sp = K._seed_args(seed)
        _lib.call("ls2_bdr_layernorm_fwd", proj.data_ptr(), bb.data_ptr(), res.data_ptr(),
                  y.data_ptr(), keep.data_ptr(), lw.data_ptr(), lb.data_ptr(), u.data_ptr(),
                  mu.data_ptr(), sg.data_ptr(), r, d, float(eps),
                  2 if (use and banked is not None) else use, sv, sp, thresh, ds,
                  _lib.dtype_code(dt), _lib.dtype_code(dt), _lib.dtype_code(sdt),
                  _lib.stream_handle())
    elif banked is not None:
        K.bias_dropout_residual(proj, bb, res, p_drop, seed, out=y,
                                mask=DropoutMask(p=p_drop, bits=keep, shape=(b, l, d)))
        K.layernorm_forward(y, lw, lb, eps, out=u, mu_out=mu, sigma_out=sg,
                            check_degenerate=False)
    else:
        K.bias_dropout_residual(proj, bb, res, p_drop, seed, out=y, bits_out=keep)
        K.layernorm_forward(y, lw, lb, eps, out=u, mu_out=mu, sigma_out=sg,
                            check_degenerate=False)
    return y, keep, mu, sg, u



def _tail_ln_fwd(proj, bias, res, p_drop, seed, ln_w, ln_b, eps, arena, stash, p, keep_tag,
                 y_tag, ln):
    """_tail_ln_core + stash: pushes keep, y, mu, sg, u (in that order); returns (y, u)."""
    y, keep, mu, sg, u = _tail_ln_core(proj, bias, res, p_drop, seed, ln_w, ln_b, eps, arena)
    stash.push(p + keep_tag, keep); stash.push(p + y_tag, y)
    stash.push(p + "mu" + ln, mu); stash.push(p + "sg" + ln, sg); stash.push(p + "u" + ln, u)
    return y, u


def _self_attention_fwd(x, w, mask, p_drop, seed, site, n_heads, eps, arena, stash, p, pre=None):
    """pre: (u1, mu1, sg1) = LN1(x) already produced by the previous layer's
    fused FFN tail (chain fusion), else LN1 runs here."""
    b, l, d = x.shape
    r, dt, hd = b * l, x.dtype, d // n_heads
    sdt = _stat_dtype(dt)
    stash.push(p + "x_in", x)
    if pre is not None:
        u1, mu1, sg1 = pre
    else:
        mu1, sg1 = arena.alloc((r,), sdt), arena.alloc((r,), sdt)
        u1 = arena.alloc((b, l, d), dt)
        K.layernorm_forward(x, _as_dt(w.ln1_w, dt), _as_dt(w.ln1_b, dt), eps, out=u1, mu_out=mu1,
                            sigma_out=sg1, check_degenerate=False)
    stash.push(p + "mu1", mu1); stash.push(p + "sg1", sg1); stash.push(p + "u1", u1)
    qkv = arena.alloc((b, l, 3 * d), dt)
    _linear(u1.view(r, d), w.wqkv, w.bqkv, qkv.view(r, 3 * d))
    stash.push(p + "qkv", qkv)
    if ATT.fused_ok(dt, l, l, hd, mask, flash=True):
        scores = ATT.alloc_state(arena, dt, b, n_heads, l, l, hd, mask, flash=True)
        ctxm = arena.alloc((b, l, d), dt)
        ATT.forward(qkv[..., :d], 3 * d, qkv[..., d:2 * d], 3 * d, qkv[..., 2 * d:], 3 * d,
                    scores, ctxm, d, b, n_heads, l, l, hd, mask, 1.0 / math.sqrt(hd))
        stash.push(p + "probs", scores)
    else:
        scores = arena.alloc((b, n_heads, l, l), dt)
        qh, kh, vh = _qkv_heads(qkv, n_heads)
        K.gemm(qh, kh, trans_b=True, out=scores, alpha=1.0 / math.sqrt(hd))
        K.softmax_forward(scores, mask=mask, out=scores)
        stash.push(p + "probs", scores)
        ctxm = arena.alloc((b, l, d), dt)
        K.gemm(scores, vh, out=_heads(ctxm, n_heads))
    stash.push(p + "ctxm", ctxm)
    proj = arena.alloc((b, l, d), dt)
    _linear(ctxm.view(r, d), w.wo, None, proj.view(r, d))
    # attention tail fused with the LayerNorm that follows it (ln2 in both layer kinds)
    y1, u2 = _tail_ln_fwd(proj, w.bo, x, p_drop, _site_seed(seed, site, 0), w.ln2_w, w.ln2_b,
                          eps, arena, stash, p, "keep1", "y1", "2")
    arena.free(proj)
    return y1, u2


# Test hook: when a dict, every FFN forward stores a copy of its ReLU bit mask
# (byte i>>3, bit i&7 of the flat [B, L, F] index) under its stash prefix, so a
# parity test can hand the GPU's ReLU decisions to the oracle (a pre-activation
# within rounding of 0 may fall on either side; see tests/test_gpu_headline.py).
RELU_TAP: dict | None = None
# Test hook: when a dict, the decoder backward stores copies of the gradient
# entering each decoder layer ("ddec", "dg5", ..., "dg0" = the layer's output
# gradient) and of each cross-attention query gradient ("dqc:dec{i}.").
GRAD_TAP: dict | None = None


def _ffn_fwd(y_in, u, w, p_drop, seed, site, k_relu, k_tail, arena, stash, p, next_ln=None):
    """FFN sublayer on the already-normalized input u = LN(y_in).

    next_ln: (w, b, eps) of the LayerNorm that consumes this layer's output (the
    next layer's ln1, or the stack's final LN): the FFN tail is then fused with
    it and (y2, (u, mu, sigma)) is returned instead of y2."""
    b, l, d = y_in.shape
    r, dt = b * l, y_in.dtype
    dff = w.w1.shape[0]
    a1 = arena.alloc((b, l, dff), dt)
    _linear(u.view(r, d), w.w1, None, a1.view(r, dff))
    z = arena.alloc((b, l, dff), dt)
    s_relu = _site_seed(seed, site, k_relu)
    banked = _bank_bits(s_relu, r * dff) if p_drop > 0.0 else None
    keep_r = banked if banked is not None else arena.alloc((_nbits(r * dff),), torch.uint8)
    relum = arena.alloc((_nbits(r * dff),), torch.uint8)
    K.bias_relu_dropout(a1, _as_dt(w.b1, dt), p_drop, s_relu, out=z, bits_out=keep_r,
                        relu_bits_out=relum,
                        mask=None if banked is None else
                        DropoutMask(p=p_drop, bits=keep_r, shape=(b, l, dff)))
    arena.free(a1)
    if RELU_TAP is not None:
        # under graph capture the copy lands in the graph's pool and is
        # refreshed by every replay
        RELU_TAP[("graph:" if torch.cuda.is_current_stream_capturing() else "") + p] = relum.clone()
    stash.push(p + "keepr", keep_r); stash.push(p + "relum", relum); stash.push(p + "z", z)
    f = arena.alloc((b, l, d), dt)
    _linear(z.view(r, dff), w.w2, None, f.view(r, d))
    s_tail = _site_seed(seed, site, k_tail)
    if next_ln is not None:
        nw, nb, neps = next_ln
        y2, keep_t, mu, sg, un = _tail_ln_core(f, w.b2, y_in, p_drop, s_tail, nw, nb, neps, arena)
        arena.free(f)
        stash.push(p + "keept", keep_t)
        return y2, (un, mu, sg)
    y2 = arena.alloc((b, l, d), dt)
    banked = _bank_bits(s_tail, r * d) if p_drop > 0.0 else None
    keep_t = banked if banked is not None else arena.alloc((_nbits(r * d),), torch.uint8)
    K.bias_dropout_residual(f, _as_dt(w.b2, dt), y_in, p_drop, s_tail, out=y2, bits_out=keep_t,
                            mask=None if banked is None else
                            DropoutMask(p=p_drop, bits=keep_t, shape=(b, l, d)))
    arena.free(f)
    stash.push(p + "keept", keep_t)
    return y2


def encoder_layer_forward(x, w: EncoderLayerWeights, mask, p_drop, seed, *, n_heads, eps=1e-5,
                          arena=None, stash=None, prefix="", site=0, strategy=None):
    """One pre-LN encoder layer; returns (y, stash).  x moves into the stash."""
    arena = arena or NullArena()
    stash = stash if stash is not None else ActivationStash()
    x = x if isinstance(x, torch.Tensor) else K.dev(x)
    y2, _ = _enc_fwd_chain(x, w, mask, p_drop, seed, n_heads, eps, arena, stash, prefix, site)
    return y2, stash


def _enc_fwd_chain(x, w, mask, p_drop, seed, n_heads, eps, arena, stash, prefix, site, pre=None,
                   next_ln=None):
    """Encoder layer inside a stack: pre = this layer's LN1 from the previous
    layer's fused tail; next_ln = the LN after this layer (fused into its FFN
    tail).  Returns (y, LN-of-y triple or None)."""
    y1, u2 = _self_attention_fwd(x, w, mask, p_drop, seed, site, n_heads, eps, arena, stash,
                                 prefix, pre=pre)
    out = _ffn_fwd(y1, u2, w, p_drop, seed, site, 1, 2, arena, stash, prefix, next_ln=next_ln)
    return out if next_ln is not None else (out, None)


def _ln_bwd_tail(sink, pp, ln, du, y_in, w_ln, mu, sg, dyo, dres, keep, p_drop, bias_name,
                 dproj) -> bool:
    """LayerNorm backward (+ dres) fused with the preceding bias+dropout+residual
    backward (ls2_layernorm_bwd_bdr): writes dyo and dproj and the ln.w / ln.b /
    bias gradients in one pass.  Returns False when the shapes need the unfused ops."""
    dt = du.dtype
    lw = _as_dt(w_ln, dt)
    if not (_fusable_rows(du, y_in, lw, dres, dyo, dproj) and y_in.dtype == dt
            and mu.dtype == torch.float32):
        return False
    b, l, d = du.shape
    r = b * l
    names = (pp + ln + ".w", pp + ln + ".b", bias_name)
    ws = _defer(sink, list(names), int(_lib._lib.ls2_layernorm_bwd_nblk(r, d)), 3, d)
    if ws is not None:                    # partials only; finished inside the narrow pass
        outs, mask, staged = [None, None, None], 0, False
    else:
        tg = [sink.target(nm) for nm in names]
        if all(t is not None for t in tg) and len({t[0].dtype for t in tg}) == 1:
            outs = [t[0] for t in tg]
            mask = sum(int(t[1]) << k for k, t in enumerate(tg))
            staged = False
        else:
            outs = [torch.empty(d, dtype=torch.float32, device=du.device) for _ in names]
            mask, staged = 0, True
        ws = _lib.context().scratch("reduce", _lib.call_i64("ls2_layernorm_bwd_ws_bytes", r, d))
    use, _, ds = K._drop_args(p_drop)
    _lib.call("ls2_layernorm_bwd_bdr", du.data_ptr(), y_in.data_ptr(), lw.data_ptr(),
              mu.data_ptr(), sg.data_ptr(), _lib.ptr(dres), dyo.data_ptr(), keep.data_ptr(),
              dproj.data_ptr(), use, ds, _lib.ptr(outs[0]), _lib.ptr(outs[1]),
              _lib.ptr(outs[2]), _lib.F32, mask, ws.data_ptr(), r, d,
              _lib.dtype_code(dt), _lib.dtype_code(dt), _lib.dtype_code(mu), _lib.stream_handle())
    if staged:
        for nm, o in zip(names, outs):
            sink.add(nm, o)
    return True


def _ffn_bwd(dy, w, stash, sink, p_drop, arena, p, pp, ln, y_in_tag, tail=None, df_in=None):
    """FFN sublayer backward.  tail=(bias_name, keep_tag): also run the preceding
    attention tail's bias+dropout+residual backward in the LayerNorm pass and
    return (dyo, dproj); otherwise return (dyo, None).  df_in: the FFN tail's
    bias+dropout backward already done (fused into the next LayerNorm's
    backward, chain fusion): its dx, with the ffn.b2 gradient already taken."""
    b, l, d = dy.shape
    r, dt = b * l, dy.dtype
    dff = w.w1.shape[0]
    keep_t = stash.pop(p + "keept") if df_in is None else None
    z = stash.pop(p + "z")
    relum = stash.pop(p + "relum")
    keep_r = stash.pop(p + "keepr")
    u = stash.pop(p + "u" + ln)
    sg = stash.pop(p + "sg" + ln)
    mu = stash.pop(p + "mu" + ln)
    y_in = stash.pop(p + y_in_tag)
    if df_in is None:
        df = arena.alloc((b, l, d), dt)
        _bdr_bwd(sink, pp + "ffn.b2", dy, keep_t, p_drop, df)
        arena.free(keep_t)
    else:
        df = df_in
    dz = arena.alloc((b, l, dff), dt)
    K.gemm(df.view(r, d), _as_dt(w.w2, dt), out=dz.view(r, dff))
    _wgrad(sink, pp + "ffn.w2", df.view(r, d), z.view(r, dff))
    arena.free(z); arena.free(df)
    da1 = arena.alloc((b, l, dff), dt)
    _brd_bwd(sink, pp + "ffn.b1", dz, keep_r, relum, p_drop, da1)
    arena.free(dz); arena.free(relum); arena.free(keep_r)
    du = arena.alloc((b, l, d), dt)
    K.gemm(da1.view(r, dff), _as_dt(w.w1, dt), out=du.view(r, d))
    _wgrad(sink, pp + "ffn.w1", da1.view(r, dff), u.view(r, d))
    arena.free(da1); arena.free(u)
    dyo = arena.alloc((b, l, d), dt)
    dproj = None
    if tail is not None:
        keep = stash.pop(p + tail[1])
        dproj = arena.alloc((b, l, d), dt)
        if not _ln_bwd_tail(sink, pp, "ln" + ln, du, y_in, getattr(w, f"ln{ln}_w"), mu, sg, dyo,
                            dy, keep, p_drop, tail[0], dproj):
            _ln_bwd(sink, pp, "ln" + ln, du, y_in, getattr(w, f"ln{ln}_w"), mu, sg, dyo, dy)
            _bdr_bwd(sink, tail[0], dyo, keep, p_drop, dproj)
        arena.free(keep)
    else:
        _ln_bwd(sink, pp, "ln" + ln, du, y_in, getattr(w, f"ln{ln}_w"), mu, sg, dyo, dy)
    arena.free(du); arena.free(mu); arena.free(sg); arena.free(y_in)
    arena.free(dy)
    return dyo, dproj


def _self_attention_bwd(dy1, w, stash, sink, n_heads, p_drop, arena, p, pp, dproj=None,
                        tail_prev=None):
    """Self-attention sublayer backward.  dproj: the attention-tail gradient when
    the caller already produced it (fused into the LayerNorm backward).
    tail_prev: (prefix, param prefix) of the layer below: its FFN tail's
    bias+dropout backward is fused into this LN1 backward, and (dx, df_prev) is
    returned instead of dx."""
    b, l, d = dy1.shape
    r, dt, hd = b * l, dy1.dtype, d // n_heads
    if dproj is None:
        keep1 = stash.pop(p + "keep1")
    ctxm = stash.pop(p + "ctxm")
    probs = stash.pop(p + "probs")
    qkv = stash.pop(p + "qkv")
    u1 = stash.pop(p + "u1")
    sg1 = stash.pop(p + "sg1")
    mu1 = stash.pop(p + "mu1")
    x_in = stash.pop(p + "x_in")
    if dproj is None:
        dproj = arena.alloc((b, l, d), dt)
        _bdr_bwd(sink, pp + "attn.bo", dy1, keep1, p_drop, dproj)
        arena.free(keep1)
    dctxm = arena.alloc((b, l, d), dt)
    K.gemm(dproj.view(r, d), _as_dt(w.wo, dt), out=dctxm.view(r, d))
    _wgrad(sink, pp + "attn.wo", dproj.view(r, d), ctxm.view(r, d))
    arena.free(dproj)
    bias_done = False
    if ATT.fused_ok(dt, l, l, hd, AttentionMask("none"), flash=True):
        dqkv = arena.alloc((b, l, 3 * d), dt)
        # the qkv bias gradient leaves the kernel as per-batch (flash: per 128-row
        # block) column partials
        part = _defer(sink, [pp + "attn.bqkv"], ATT.bias_rows(b, l, l), 1, 3 * d)
        ATT.backward(qkv[..., :d], 3 * d, qkv[..., d:2 * d], 3 * d, qkv[..., 2 * d:], 3 * d,
                     probs, dctxm, d, dqkv[..., :d], 3 * d, dqkv[..., d:2 * d], 3 * d,
                     dqkv[..., 2 * d:], 3 * d, b, n_heads, l, l, hd, 1.0 / math.sqrt(hd),
                     colsums=None if part is None else
                     ((part, 0, 3 * d), (part, d, 3 * d), (part, 2 * d, 3 * d)),
                     o=ctxm, ldo=d)
        bias_done = part is not None
        arena.free(probs); arena.free(dctxm); arena.free(qkv); arena.free(ctxm)
    else:
        dctx = _heads(dctxm, n_heads)
        qh, kh, vh = _qkv_heads(qkv, n_heads)
        dscores = arena.alloc((b, n_heads, l, l), dt)
        K.gemm(dctx, vh, trans_b=True, out=dscores)
        G.softmax_backward(dscores, SoftmaxCache(probs), out=dscores,
                           out_scale=1.0 / math.sqrt(hd))
        dqkv = arena.alloc((b, l, 3 * d), dt)
        dq, dk, dv = _qkv_heads(dqkv, n_heads)
        K.gemm(dscores, kh, out=dq)
        K.gemm(dscores, qh, trans_a=True, out=dk)
        K.gemm(probs, dctx, trans_a=True, out=dv)
        arena.free(dscores); arena.free(probs); arena.free(dctxm); arena.free(qkv)
        arena.free(ctxm)
    du1 = arena.alloc((b, l, d), dt)
    K.gemm(dqkv.view(r, 3 * d), _as_dt(w.wqkv, dt), out=du1.view(r, d))
    _wgrad(sink, pp + "attn.wqkv", dqkv.view(r, 3 * d), u1.view(r, d))
    if not bias_done:
        _colsum_grad(sink, pp + "attn.bqkv", dqkv.view(r, 3 * d))
    arena.free(dqkv); arena.free(u1)
    dx = arena.alloc((b, l, d), dt)
    if tail_prev is None:
        _ln_bwd(sink, pp, "ln1", du1, x_in, w.ln1_w, mu1, sg1, dx, dy1)
        arena.free(du1); arena.free(mu1); arena.free(sg1); arena.free(x_in)
        arena.free(dy1)
        return dx
    df_prev = _ln_bwd_chain(sink, pp, "ln1", du1, x_in, w.ln1_w, mu1, sg1, dx, dy1, stash,
                            tail_prev, p_drop, arena)
    arena.free(du1); arena.free(mu1); arena.free(sg1); arena.free(x_in)
    arena.free(dy1)
    return dx, df_prev


def _ln_bwd_chain(sink, pp, ln, du, x_in, w_ln, mu, sg, dx, dres, stash, tail_prev, p_drop, arena):
    """LayerNorm backward fused with the FFN-tail bias+dropout backward of the
    layer below (tail_prev = its (prefix, param prefix)): writes dx and returns
    that layer's df (its ffn.b2 gradient taken here)."""
    prev_p, prev_pp = tail_prev
    keep_prev = stash.pop(prev_p + "keept")
    b, l, d = dx.shape
    df_prev = arena.alloc((b, l, d), dx.dtype)
    if not _ln_bwd_tail(sink, pp, ln, du, x_in, w_ln, mu, sg, dx, dres, keep_prev, p_drop,
                        prev_pp + "ffn.b2", df_prev):
        _ln_bwd(sink, pp, ln, du, x_in, w_ln, mu, sg, dx, dres)
        _bdr_bwd(sink, prev_pp + "ffn.b2", dx, keep_prev, p_drop, df_prev)
    arena.free(keep_prev)
    return df_prev


def encoder_layer_backward(dy, w: EncoderLayerWeights, stash: ActivationStash, sink: GradSink, *,
                           n_heads, p_drop, arena=None, prefix="", param_prefix="", df_in=None,
                           tail_prev=None):
    """Backward of one encoder layer. Takes ownership of dy, returns dx
    ((dx, df_prev) with tail_prev; df_in / tail_prev: chain fusion, see
    _ffn_bwd / _self_attention_bwd)."""
    arena = arena or NullArena()
    dy = dy if isinstance(dy, torch.Tensor) else K.dev(dy)
    dy1, dproj = _ffn_bwd(dy, w, stash, sink, p_drop, arena, prefix, param_prefix, "2", "y1",
                          tail=(param_prefix + "attn.bo", "keep1"), df_in=df_in)
    return _self_attention_bwd(dy1, w, stash, sink, n_heads, p_drop, arena, prefix, param_prefix,
                               dproj=dproj, tail_prev=tail_prev)


# ---------------------------------------------------------------------------
# decoder layer (F/model.py:517-775)
# ---------------------------------------------------------------------------

def decoder_layer_forward(x, w: DecoderLayerWeights, kv, self_mask, cross_mask, p_drop, seed, *,
                          n_heads, eps=1e-5, arena=None, stash=None, prefix="", site=0,
                          strategy=None, pre=None, next_ln=None):
    """One pre-LN decoder layer consuming precomputed (K_i, V_i).

    pre / next_ln: chain fusion inside a stack (see _enc_fwd_chain); with
    next_ln the return value is (y, stash, LN-of-y triple)."""
    arena = arena or NullArena()
    stash = stash if stash is not None else ActivationStash()
    x = x if isinstance(x, torch.Tensor) else K.dev(x)
    k_i, v_i = kv
    b, l, d = x.shape
    r, dt, hd = b * l, x.dtype, d // n_heads
    ls = k_i.shape[1]
    p = prefix
    y1, u2 = _self_attention_fwd(x, w, self_mask, p_drop, seed, site, n_heads, eps, arena, stash,
                                 p, pre=pre)
    qc = arena.alloc((b, l, d), dt)
    _linear(u2.view(r, d), w.cross_wq, w.cross_bq, qc.view(r, d))
    stash.push(p + "qc", qc)
    if ATT.fused_ok(dt, l, ls, hd, cross_mask) and k_i.dtype == dt and v_i.dtype == dt:
        scores_x = ATT.alloc_state(arena, dt, b, n_heads, l, ls, hd, cross_mask)
        ctxm_x = arena.alloc((b, l, d), dt)
        ATT.forward(qc, d, k_i, k_i.stride(1), v_i, v_i.stride(1), scores_x, ctxm_x, d, b,
                    n_heads, l, ls, hd, cross_mask, 1.0 / math.sqrt(hd))
        stash.push(p + "probs_x", scores_x)
    else:
        scores_x = arena.alloc((b, n_heads, l, ls), dt)
        K.gemm(_heads(qc, n_heads), _heads(_as_dt(k_i, dt), n_heads), trans_b=True,
               out=scores_x, alpha=1.0 / math.sqrt(hd))
        K.softmax_forward(scores_x, mask=cross_mask, out=scores_x)
        stash.push(p + "probs_x", scores_x)
        ctxm_x = arena.alloc((b, l, d), dt)
        K.gemm(scores_x, _heads(_as_dt(v_i, dt), n_heads), out=_heads(ctxm_x, n_heads))
    stash.push(p + "ctxm_x", ctxm_x)
    proj_x = arena.alloc((b, l, d), dt)
    _linear(ctxm_x.view(r, d), w.cross_wo, None, proj_x.view(r, d))
    y2, u3 = _tail_ln_fwd(proj_x, w.cross_bo, y1, p_drop, _site_seed(seed, site, 1), w.ln3_w,
                          w.ln3_b, eps, arena, stash, p, "keep2", "y2", "3")
    arena.free(proj_x)
    if next_ln is not None:
        y3, tri = _ffn_fwd(y2, u3, w, p_drop, seed, site, 2, 3, arena, stash, p, next_ln=next_ln)
        return y3, stash, tri
    y3 = _ffn_fwd(y2, u3, w, p_drop, seed, site, 2, 3, arena, stash, p)
    return y3, stash


def decoder_layer_backward(dy, w: DecoderLayerWeights, kv, stash: ActivationStash, sink: GradSink,
                           *, n_heads, p_drop, arena=None, prefix="", param_prefix="",
                           dkv_out=None, kv_colsum=None, df_in=None, tail_prev=None):
    """Backward of one decoder layer; returns (dx, dK_i, dV_i).

    dkv_out: optional (dK_i, dV_i) destination views (slices of the packed
    cross-K/V gradient buffer) so packed_kv_backward needs no gather copy.
    kv_colsum: optional (partial buffer, K column, V column, row pitch): the
    fused attention backward leaves this layer's share of the packed cross-K/V
    bias gradient there."""
    arena = arena or NullArena()
    dy = dy if isinstance(dy, torch.Tensor) else K.dev(dy)
    k_i, v_i = kv
    b, l, d = dy.shape
    r, dt, hd = b * l, dy.dtype, d // n_heads
    ls = k_i.shape[1]
    p, pp = prefix, param_prefix
    dy2, dproj_x = _ffn_bwd(dy, w, stash, sink, p_drop, arena, p, pp, "3", "y2",
                            tail=(pp + "cross.bo", "keep2"), df_in=df_in)
    ctxm_x = stash.pop(p + "ctxm_x")
    probs_x = stash.pop(p + "probs_x")
    qc = stash.pop(p + "qc")
    u2 = stash.pop(p + "u2")
    sg2 = stash.pop(p + "sg2")
    mu2 = stash.pop(p + "mu2")
    dctxm_x = arena.alloc((b, l, d), dt)
    K.gemm(dproj_x.view(r, d), _as_dt(w.cross_wo, dt), out=dctxm_x.view(r, d))
    _wgrad(sink, pp + "cross.wo", dproj_x.view(r, d), ctxm_x.view(r, d))
    arena.free(dproj_x); arena.free(ctxm_x)
    cross_bias_done = False
    if ATT.fused_ok(dt, l, ls, hd, AttentionMask("none")) and k_i.dtype == dt and \
            v_i.dtype == dt and (dkv_out is None or dkv_out[0].dtype == dt):
        dqc = arena.alloc((b, l, d), dt)
        if dkv_out is not None:
            dk_i, dv_i = dkv_out
        else:
            dk_i, dv_i = arena.alloc((b, ls, d), dt), arena.alloc((b, ls, d), dt)
        part_q = _defer(sink, [pp + "cross.bq"], b, 1, d)
        kvcs = (None, None)
        if kv_colsum is not None and dkv_out is not None:
            kbuf, kcol, vcol, kld = kv_colsum
            kvcs = ((kbuf, kcol, kld), (kbuf, vcol, kld))
        ATT.backward(qc, d, k_i, k_i.stride(1), v_i, v_i.stride(1), probs_x, dctxm_x, d,
                     dqc, d, dk_i, dk_i.stride(1), dv_i, dv_i.stride(1), b, n_heads, l, ls, hd,
                     1.0 / math.sqrt(hd),
                     colsums=(None if part_q is None else (part_q, 0, d), kvcs[0], kvcs[1]))
        cross_bias_done = part_q is not None
        arena.free(probs_x); arena.free(dctxm_x); arena.free(qc)
    else:
        dctx_x = _heads(dctxm_x, n_heads)
        kh, vh = _heads(_as_dt(k_i, dt), n_heads), _heads(_as_dt(v_i, dt), n_heads)
        dscores_x = arena.alloc((b, n_heads, l, ls), dt)
        K.gemm(dctx_x, vh, trans_b=True, out=dscores_x)
        G.softmax_backward(dscores_x, SoftmaxCache(probs_x), out=dscores_x,
                           out_scale=1.0 / math.sqrt(hd))
        dqc = arena.alloc((b, l, d), dt)
        K.gemm(dscores_x, kh, out=_heads(dqc, n_heads))
        if dkv_out is not None:
            dk_i, dv_i = dkv_out
        else:
            dk_i, dv_i = arena.alloc((b, ls, d), dt), arena.alloc((b, ls, d), dt)
        K.gemm(dscores_x, _heads(qc, n_heads), trans_a=True, out=_heads(dk_i, n_heads))
        K.gemm(probs_x, dctx_x, trans_a=True, out=_heads(dv_i, n_heads))
        arena.free(dscores_x); arena.free(probs_x); arena.free(dctxm_x); arena.free(qc)
    if GRAD_TAP is not None:
        GRAD_TAP["dqc:" + p] = dqc.clone()
    du2 = arena.alloc((b, l, d), dt)
    K.gemm(dqc.view(r, d), _as_dt(w.cross_wq, dt), out=du2.view(r, d))
    _wgrad(sink, pp + "cross.wq", dqc.view(r, d), u2.view(r, d))
    if not cross_bias_done:
        _colsum_grad(sink, pp + "cross.bq", dqc.view(r, d))
    arena.free(dqc); arena.free(u2)
    y1 = stash.pop(p + "y1")
    keep1 = stash.pop(p + "keep1")
    dy1 = arena.alloc((b, l, d), dt)
    dproj = arena.alloc((b, l, d), dt)
    if not _ln_bwd_tail(sink, pp, "ln2", du2, y1, w.ln2_w, mu2, sg2, dy1, dy2, keep1, p_drop,
                        pp + "attn.bo", dproj):
        _ln_bwd(sink, pp, "ln2", du2, y1, w.ln2_w, mu2, sg2, dy1, dy2)
        _bdr_bwd(sink, pp + "attn.bo", dy1, keep1, p_drop, dproj)
    arena.free(keep1)
    arena.free(du2); arena.free(mu2); arena.free(sg2); arena.free(y1)
    arena.free(dy2)
    if tail_prev is not None:
        dx, df_prev = _self_attention_bwd(dy1, w, stash, sink, n_heads, p_drop, arena, p, pp,
                                          dproj=dproj, tail_prev=tail_prev)
        return dx, dk_i, dv_i, df_prev
    dx = _self_attention_bwd(dy1, w, stash, sink, n_heads, p_drop, arena, p, pp, dproj=dproj)
    return dx, dk_i, dv_i


# ---------------------------------------------------------------------------
# full model (F/model.py:782-1003)
# ---------------------------------------------------------------------------

@dataclass
class Batch:
    src: object
    tgt_in: object
    tgt_out: object
    src_len: object
    pad_id: int = 0


class ModelOutput:
    """(loss_sum, token_count, correct); device-resident until first read."""

    def __init__(self, out3: torch.Tensor):
        self.out3 = out3
        self._host = None

    def _h(self):
        if self._host is None:
            self._host = self.out3.detach().cpu().numpy()
        return self._host

    @property
    def loss_sum(self) -> float:
        return float(self._h()[0])

    @property
    def token_count(self) -> int:
        return int(self._h()[1])

    @property
    def correct(self) -> int:
        return int(self._h()[2])

    @property
    def loss_per_token(self) -> float:
        return self.loss_sum / max(self.token_count, 1)

    @property
    def accuracy(self) -> float:
        return self.correct / max(self.token_count, 1)


def validate_batch(batch: Batch, cfg: ModelConfig):
    """Host-side checks the reference raises before compute."""
    src = np.asarray(batch.src)
    tin = np.asarray(batch.tgt_in)
    tout = np.asarray(batch.tgt_out)
    lens = np.asarray(batch.src_len)
    for name, t in (("src", src), ("tgt_in", tin)):
        if t.ndim != 2:
            raise ShapeMismatch(f"{name} must be [B, L]")
        if t.shape[1] > cfg.max_len:
            raise SequenceTooLong(f"sequence length {t.shape[1]} > max_len {cfg.max_len}")
        if t.size and (t.min() < 0 or t.max() >= cfg.vocab):
            raise TokenOutOfRange(f"token ids outside [0, {cfg.vocab})")
    valid = tout[tout != batch.pad_id]
    if valid.size and (valid.min() < 0 or valid.max() >= cfg.vocab):
        raise TokenOutOfRange(f"target outside [0, {cfg.vocab})")
    if lens.min() < 1 or lens.max() > src.shape[1]:
        raise ShapeMismatch("padding valid length outside [1, Lk]")


class Transformer:
    """Fused-graph encoder-decoder with a hand-wired forward/backward."""

    def __init__(self, cfg: ModelConfig, compute_dtype: torch.dtype | None = None):
        self.cfg = cfg
        self.param_names = [name for name, _ in param_spec(cfg)]
        self.compute_dtype = compute_dtype
        self._sin = None
        self._seeds: SeedTable | None = None

    def param_spec(self):
        return param_spec(self.cfg)

    def init_params(self, seed: int):
        return init_params(self.cfg, seed)

    def _positional(self, params, dtype):
        if self.cfg.learned_positional:
            return params["pos_emb"]
        if self._sin is None or self._sin.dtype != dtype:
            self._sin = sinusoidal_table(self.cfg.max_len, self.cfg.d_model, dtype)
        return self._sin

    def packed_weights(self, params) -> PackedCrossWeights:
        return PackedCrossWeights(w=params["cross_kv.w"], b=params["cross_kv.b"],
                                  n_layers=self.cfg.n_dec, d=self.cfg.d_model)

    def act_dtype(self, params) -> torch.dtype:
        if self.compute_dtype is not None:
            return self.compute_dtype
        dt = params["tok_emb"].dtype if isinstance(params["tok_emb"], torch.Tensor) else \
            K.compute_dtype(params["tok_emb"])
        return dt if dt in (torch.float16, torch.bfloat16, torch.float32, torch.float64) else torch.float32

    def seed_table(self, device) -> SeedTable:
        if self._seeds is None:
            self._seeds = SeedTable(device)
        return self._seeds

    def register_seeds(self, seeds: SeedTable, seed: int, step: int, p_drop: float):
        """Per-site dropout seeds of one step in a fixed slot order
        (F/model.py:868-898 seed derivations: (seed,step,0..3), then site, k)."""
        cfg = self.cfg
        seeds.reset()
        seeds.set_step(step)
        s_src = seeds.slot(derive_seed(seed, step, 0))
        enc_seed = _LayerSeed(seeds, derive_seed(seed, step, 1))
        s_tgt = seeds.slot(derive_seed(seed, step, 2))
        dec_seed = _LayerSeed(seeds, derive_seed(seed, step, 3))
        if p_drop > 0.0:
            for i in range(cfg.n_enc):
                for k in range(3):
                    enc_seed.site(i, k)
            for i in range(cfg.n_dec):
                for k in range(4):
                    dec_seed.site(i, k)
        return s_src, enc_seed, s_tgt, dec_seed

    def forward_backward(self, params, batch: Batch, *, p_drop=0.0, alpha=0.0, seed=0, step=0,
                         arena=None, sink: GradSink | None = None, compute_grads=True,
                         grad_scale=1.0, trace=None, strategy=None, capture: dict | None = None,
                         validate: bool = True, upload_seeds: bool = True,
                         masks: MaskBank | None = None) -> ModelOutput:
        """Run one batch end to end; gradients go into `sink`.

        grad_scale multiplies the criterion gradient.  compute_grads=False is a
        pure forward (evaluation).  capture receives "logq" (debug hook).
        masks: a MaskBank drawing every forward dropout site in one launch."""
        global _MASKS
        if masks is None:
            return self._forward_backward(params, batch, p_drop=p_drop, alpha=alpha, seed=seed,
                                          step=step, arena=arena, sink=sink,
                                          compute_grads=compute_grads, grad_scale=grad_scale,
                                          trace=trace, strategy=strategy, capture=capture,
                                          validate=validate, upload_seeds=upload_seeds)
        _MASKS = masks
        try:
            return self._forward_backward(params, batch, p_drop=p_drop, alpha=alpha, seed=seed,
                                          step=step, arena=arena, sink=sink,
                                          compute_grads=compute_grads, grad_scale=grad_scale,
                                          trace=trace, strategy=strategy, capture=capture,
                                          validate=validate, upload_seeds=upload_seeds)
        finally:
            masks.active = False
            _MASKS = None

    def _mask_sites(self, s_src, enc_seed, s_tgt, dec_seed, ts: int, tt: int):
        """(seed slot, elements) of every forward dropout site, in consumption
        order, for ts source and tt target tokens."""
        d, f = self.cfg.d_model, self.cfg.d_ff
        slot = lambda t: t.storage_offset()      # noqa: E731
        sites = [(slot(s_src), ts * d, "src")]
        for i in range(self.cfg.n_enc):
            g = f"enc{i}"
            sites += [(slot(enc_seed.site(i, 0)), ts * d, g), (slot(enc_seed.site(i, 1)), ts * f, g),
                      (slot(enc_seed.site(i, 2)), ts * d, g)]
        sites.append((slot(s_tgt), tt * d, "tgt"))
        for i in range(self.cfg.n_dec):
            g = f"dec{i}"
            sites += [(slot(dec_seed.site(i, 0)), tt * d, g), (slot(dec_seed.site(i, 1)), tt * d, g),
                      (slot(dec_seed.site(i, 2)), tt * f, g), (slot(dec_seed.site(i, 3)), tt * d, g)]
        return sites

    def _forward_backward(self, params, batch: Batch, *, p_drop, alpha, seed, step, arena, sink,
                          compute_grads, grad_scale, trace, strategy, capture, validate,
                          upload_seeds) -> ModelOutput:
        cfg = self.cfg
        ctx = _lib.context()
        arena = arena or NullArena(ctx.device)
        stash = ActivationStash()
        sink = GradSink() if sink is None else sink
        if isinstance(sink, _ViewSink):
            sink.arena = arena
        emit = trace.append if trace is not None else (lambda ev: None)
        if validate:
            validate_batch(batch, cfg)
        src = K.dev(batch.src, torch.int64)
        tgt_in = K.dev(batch.tgt_in, torch.int64)
        tgt_out = K.dev(batch.tgt_out, torch.int64).reshape(-1)
        src_len = K.dev(batch.src_len, torch.int64)
        b, ls = src.shape
        lt = tgt_in.shape[1]
        d, n, v = cfg.d_model, cfg.n_heads, cfg.vocab
        params = {k: (t if isinstance(t, torch.Tensor) else K.dev(t)) for k, t in params.items()}
        dt = self.act_dtype(params)
        sdt = _stat_dtype(dt)
        emb_cfg = EmbeddingConfig(scale=cfg.scale, vocab=v, max_len=cfg.max_len,
                                  learned_positional=cfg.learned_positional)
        tok_emb = _as_dt(params["tok_emb"], dt)
        pos = _as_dt(self._positional(params, dt), dt)
        enc_mask = AttentionMask("padding", src_len)
        dec_mask = AttentionMask("causal")
        cross_mask = AttentionMask("padding", src_len)

        seeds = self.seed_table(ctx.device)
        s_src, enc_seed, s_tgt, dec_seed = self.register_seeds(seeds, seed, step, p_drop)
        if p_drop > 0.0 and upload_seeds:
            seeds.upload()
        bank = _MASKS
        if bank is not None and p_drop > 0.0 and dt != torch.float64:
            # every forward dropout site of the step in one launch (a no-op on the
            # device when the bits were drawn beside the previous step's Adam)
            bank.prepare(lambda ts, tt: self._mask_sites(s_src, enc_seed, s_tgt, dec_seed, ts, tt),
                         b * ls, b * lt, K._drop_args(p_drop)[1])
            bank.generate(seeds.dev, stamp=bank.stamp, want=seeds.step_slot())
            bank.active = True
            arena = _BankArena(arena, bank)

        # --- forward: encoder ---
        h = arena.alloc((b, ls, d), dt)
        keep_src = _bank_bits(s_src, b * ls * d) if p_drop > 0.0 else None
        banked = keep_src is not None
        if not banked:
            keep_src = arena.alloc((_nbits(b * ls * d),), torch.uint8)
        K.embedding_forward(tok_emb, pos, src, emb_cfg, p_drop, s_src, out=h, bits_out=keep_src,
                            validate=False,
                            mask=DropoutMask(p=p_drop, bits=keep_src, shape=(b, ls, d)) if banked
                            else None)
        stash.push("src_keep", keep_src)
        enc_w = [EncoderLayerWeights.from_params(params, f"enc{i}.") for i in range(cfg.n_enc)]
        chain = CHAIN_FUSE and cfg.n_enc > 0
        pre = None
        for i in range(cfg.n_enc):
            if chain:
                nxt = (enc_w[i + 1].ln1_w, enc_w[i + 1].ln1_b) if i + 1 < cfg.n_enc else \
                    (params["enc_ln.w"], params["enc_ln.b"])
                h, pre = _enc_fwd_chain(h, enc_w[i], enc_mask, p_drop, enc_seed, n, cfg.eps, arena,
                                        stash, f"enc{i}.", i, pre=pre, next_ln=(*nxt, cfg.eps))
            else:
                h, _ = encoder_layer_forward(h, enc_w[i], enc_mask, p_drop, enc_seed, n_heads=n,
                                             eps=cfg.eps, arena=arena, stash=stash, prefix=f"enc{i}.",
                                             site=i)
        stash.push("enc_ln_in", h)
        if chain:
            enc_out, mu_e, sg_e = pre
        else:
            mu_e, sg_e = arena.alloc((b * ls,), sdt), arena.alloc((b * ls,), sdt)
            enc_out = arena.alloc((b, ls, d), dt)
            K.layernorm_forward(h, _as_dt(params["enc_ln.w"], dt), _as_dt(params["enc_ln.b"], dt),
                                cfg.eps, out=enc_out, mu_out=mu_e, sigma_out=sg_e,
                                check_degenerate=False)
        stash.push("enc_ln_mu", mu_e); stash.push("enc_ln_sg", sg_e)
        stash.push("enc_out", enc_out)
        pw = self.packed_weights(params)
        kv_pairs, kv_buf = packed_kv_forward(enc_out, pw, arena=arena)

        # --- forward: decoder ---
        g = arena.alloc((b, lt, d), dt)
        keep_tgt = _bank_bits(s_tgt, b * lt * d) if p_drop > 0.0 else None
        banked = keep_tgt is not None
        if not banked:
            keep_tgt = arena.alloc((_nbits(b * lt * d),), torch.uint8)
        K.embedding_forward(tok_emb, pos, tgt_in, emb_cfg, p_drop, s_tgt, out=g,
                            bits_out=keep_tgt, validate=False,
                            mask=DropoutMask(p=p_drop, bits=keep_tgt, shape=(b, lt, d)) if banked
                            else None)
        stash.push("tgt_keep", keep_tgt)
        dec_w = [DecoderLayerWeights.from_params(params, f"dec{i}.") for i in range(cfg.n_dec)]
        dchain = CHAIN_FUSE and cfg.n_dec > 0
        pre = None
        for i in range(cfg.n_dec):
            if dchain:
                nxt = (dec_w[i + 1].ln1_w, dec_w[i + 1].ln1_b) if i + 1 < cfg.n_dec else \
                    (params["dec_ln.w"], params["dec_ln.b"])
                g, _, pre = decoder_layer_forward(g, dec_w[i], kv_pairs[i], dec_mask, cross_mask,
                                                  p_drop, dec_seed, n_heads=n, eps=cfg.eps,
                                                  arena=arena, stash=stash, prefix=f"dec{i}.",
                                                  site=i, pre=pre, next_ln=(*nxt, cfg.eps))
            else:
                g, _ = decoder_layer_forward(g, dec_w[i], kv_pairs[i], dec_mask, cross_mask,
                                             p_drop, dec_seed, n_heads=n, eps=cfg.eps, arena=arena,
                                             stash=stash, prefix=f"dec{i}.", site=i)
        stash.push("dec_ln_in", g)
        if dchain:
            dec_out, mu_d, sg_d = pre
        else:
            mu_d, sg_d = arena.alloc((b * lt,), sdt), arena.alloc((b * lt,), sdt)
            dec_out = arena.alloc((b, lt, d), dt)
            K.layernorm_forward(g, _as_dt(params["dec_ln.w"], dt), _as_dt(params["dec_ln.b"], dt),
                                cfg.eps, out=dec_out, mu_out=mu_d, sigma_out=sg_d,
                                check_degenerate=False)
        stash.push("dec_ln_mu", mu_d); stash.push("dec_ln_sg", sg_d)
        stash.push("dec_out", dec_out)

        # --- criterion: one fused pass -> loss/count/correct (+ dlogits in place) ---
        proj_w = tok_emb if cfg.tie_embeddings else _as_dt(params["out_proj.w"], dt)
        rt = b * lt
        logits = arena.alloc((rt, v), dt)
        K.gemm(dec_out.view(rt, d), proj_w, trans_b=True, out=logits)
        row_stats = arena.alloc((2 * rt,), torch.float64)
        out3 = torch.empty(3, dtype=torch.float64, device=ctx.device)
        logq = None
        if capture is not None:
            logq = torch.empty((rt, v), dtype=dt, device=ctx.device)
        if dt == torch.float64:
            self._criterion_f64(logits, tgt_out, out3, alpha, batch.pad_id, grad_scale,
                                compute_grads, logq)
        else:
            _lib.call("ls2_criterion_fused", logits.data_ptr(), tgt_out.data_ptr(),
                      logits.data_ptr() if compute_grads else None, _lib.ptr(logq),
                      row_stats.data_ptr(), out3.data_ptr(), None, rt, v, float(alpha),
                      int(batch.pad_id), 1, float(grad_scale), _lib.dtype_code(logits),
                      _lib.stream_handle())
        arena.free(row_stats)
        if isinstance(sink, _ViewSink):
            sink.totals = out3            # the exchange all-reduces these first
        out = ModelOutput(out3)
        if capture is not None:
            capture["logq"] = logq.view(b, lt, v)
        if not compute_grads:
            stash.drain(arena)
            arena.free(kv_buf)
            arena.free(logits)
            return out

        # --- backward: output projection ---
        # weight-gradient GEMMs go through the sink's lane (engine path: batched
        # across layers); frees of the buffers they read are held until it flushes
        main_arena = arena
        lane, arena, join = _open_lane(sink, arena, dt)
        dlogits = logits
        dec_out = stash.pop("dec_out")
        ddec = arena.alloc((b, lt, d), dt)
        K.gemm(dlogits, proj_w, out=ddec.view(rt, d))
        _wgrad(sink, "tok_emb" if cfg.tie_embeddings else "out_proj.w", dlogits,
               dec_out.view(rt, d))
        arena.free(dlogits); arena.free(dec_out)
        sg_d = stash.pop("dec_ln_sg"); mu_d = stash.pop("dec_ln_mu")
        g_in = stash.pop("dec_ln_in")
        dg = arena.alloc((b, lt, d), dt)
        nd = cfg.n_dec
        df = None
        if dchain:     # fused with the last decoder layer's FFN-tail backward
            df = _ln_bwd_chain(sink, "", "dec_ln", ddec, g_in, params["dec_ln.w"], mu_d, sg_d, dg,
                               None, stash, (f"dec{nd - 1}.", f"dec{nd - 1}."), p_drop, arena)
        else:
            _ln_bwd(sink, "", "dec_ln", ddec, g_in, params["dec_ln.w"], mu_d, sg_d, dg, None)
        if GRAD_TAP is not None:
            GRAD_TAP["ddec"] = ddec.clone()
            GRAD_TAP[f"dg{cfg.n_dec}"] = dg.clone()
        arena.free(ddec); arena.free(mu_d); arena.free(sg_d); arena.free(g_in)
        _ready(sink, "dec_ln.", "out_proj.")

        # --- backward: decoder stack; dK_i/dV_i land in one packed buffer ---
        dkv = arena.alloc((b, ls, 2 * cfg.n_dec * d), dt)
        dks: list = [None] * nd
        dvs: list = [None] * nd
        # the packed cross-K/V bias gradient as per-batch partials left by the
        # fused attention backward of every decoder layer (its own columns)
        kvpart = _defer(sink, ["cross_kv.b"], b, 1, 2 * nd * d) \
            if ATT.fused_ok(dt, lt, ls, d // n, AttentionMask("none")) else None
        for i in reversed(range(nd)):
            dest = (dkv[..., i * d:(i + 1) * d], dkv[..., (nd + i) * d:(nd + i + 1) * d])
            tp = (f"dec{i - 1}.", f"dec{i - 1}.") if (dchain and i > 0) else None
            res = decoder_layer_backward(
                dg, dec_w[i], kv_pairs[i], stash, sink, n_heads=n, p_drop=p_drop, arena=arena,
                prefix=f"dec{i}.", param_prefix=f"dec{i}.", dkv_out=dest,
                kv_colsum=None if kvpart is None else (kvpart, i * d, (nd + i) * d, 2 * nd * d),
                df_in=df, tail_prev=tp)
            if tp is not None:
                dg, dks[i], dvs[i], df = res
            else:
                (dg, dks[i], dvs[i]), df = res, None
            if GRAD_TAP is not None:
                GRAD_TAP[f"dg{i}"] = dg.clone()
            join()
            _ready(sink, f"dec{i}.")
            emit(("dec_layer_backward_done", i))
        keep_tgt = stash.pop("tgt_keep")
        self._embedding_grads(sink, dg, tgt_in, keep_tgt, p_drop, emb_cfg)
        arena.free(dg); arena.free(keep_tgt)
        arena.free(kv_buf)

        # --- backward: packed cross K/V (only now is the enc grad legal) ---
        enc_out = stash.pop("enc_out")
        denc, _, _ = packed_kv_backward(dks, dvs, enc_out, pw, arena=arena, packed=dkv, sink=sink,
                                        bias_done=kvpart is not None)
        emit(("enc_out_grad_emitted",))
        arena.free(dkv)
        arena.free(enc_out)
        sg_e = stash.pop("enc_ln_sg"); mu_e = stash.pop("enc_ln_mu")
        h_in = stash.pop("enc_ln_in")
        dh = arena.alloc((b, ls, d), dt)
        df = None
        if chain:      # fused with the last encoder layer's FFN-tail backward
            ne = cfg.n_enc
            df = _ln_bwd_chain(sink, "", "enc_ln", denc, h_in, params["enc_ln.w"], mu_e, sg_e, dh,
                               None, stash, (f"enc{ne - 1}.", f"enc{ne - 1}."), p_drop, arena)
        else:
            _ln_bwd(sink, "", "enc_ln", denc, h_in, params["enc_ln.w"], mu_e, sg_e, dh, None)
        arena.free(denc); arena.free(mu_e); arena.free(sg_e); arena.free(h_in)
        join()
        _ready(sink, "cross_kv.", "enc_ln.")
        for i in reversed(range(cfg.n_enc)):
            tp = (f"enc{i - 1}.", f"enc{i - 1}.") if (chain and i > 0) else None
            res = encoder_layer_backward(dh, enc_w[i], stash, sink, n_heads=n, p_drop=p_drop,
                                         arena=arena, prefix=f"enc{i}.", param_prefix=f"enc{i}.",
                                         df_in=df, tail_prev=tp)
            dh, df = res if tp is not None else (res, None)
            join()
            _ready(sink, f"enc{i}.")
        keep_src = stash.pop("src_keep")
        self._embedding_grads(sink, dh, src, keep_src, p_drop, emb_cfg)
        arena.free(dh); arena.free(keep_src)
        join()
        _close_lane(sink, lane)
        _ready(sink, None)
        arena = main_arena
        if len(stash):
            raise ShapeMismatch(f"activation stash leaked {len(stash)} entries")
        # deferred gradient partials are consumed by the engine's narrow pass, which
        # is stream-ordered after this step and before any reuse of the arena
        for buf in getattr(sink, "deferred_buffers", lambda: [])():
            arena.free(buf)
        return out

    def _embedding_grads(self, sink, dy, tokens, keep_bits, p_drop, emb_cfg):
        mask = DropoutMask(p=p_drop, bits=keep_bits, shape=tuple(dy.shape))
        te = sink.target("tok_emb")
        tp = sink.target("pos_emb") if emb_cfg.learned_positional else None
        if te is not None and (tp is not None or not emb_cfg.learned_positional):
            ev, ebeta = te
            if not ebeta:
                ev.zero_()
            G.embedding_backward(dy, tokens, mask, emb_cfg, dE_out=ev,
                                 dP_out=None if tp is None else tp[0],
                                 beta_pos=0 if tp is None else tp[1], validate=False)
            return
        de, dp = G.embedding_backward(dy, tokens, mask, emb_cfg, validate=False)
        sink.add("tok_emb", de)
        if dp is not None:
            sink.add("pos_emb", dp)

    def _criterion_f64(self, logits, tgt_out, out3, alpha, pad_id, grad_scale, compute_grads,
                       logq_out):
        """float64 path (finite-difference checks): reference-API kernels."""
        lq = K.log_softmax_forward(logits)
        loss, count = K.ls_cross_entropy_forward(lq, tgt_out, alpha, pad_id)
        ok = tgt_out != pad_id
        correct = int((lq.argmax(dim=-1)[ok] == tgt_out[ok]).sum())
        out3.copy_(torch.tensor([loss, count, correct], dtype=torch.float64))
        if logq_out is not None:
            logq_out.copy_(lq)
        if compute_grads:
            G.ls_cross_entropy_backward(torch.exp(lq), tgt_out, alpha, pad_id,
                                        grad_scale=grad_scale, out=logits, check=False)


def transformer_forward_backward(cfg: ModelConfig, params, batch: Batch, **kwargs):
    """Functional wrapper: run one batch and return (output, grads dict)."""
    sink = kwargs.pop("sink", None) or GradSink()
    out = Transformer(cfg).forward_backward(params, batch, sink=sink, **kwargs)
    return out, sink.store


class EncoderMLM(Transformer):
    """BERT-shaped encoder with a tied masked-LM criterion (BASELINE.json
    configs[3]): not a reference model, composed from the
    reference's own pieces — embedding (F/kernels.py:203-228), pre-LN encoder
    layers (F/model.py:335-510), final LayerNorm, tied output projection and
    the label-smoothed criterion (F/model.py:908-939).  Non-MLM positions carry
    the pad target, so the criterion skips them (count = MLM tokens).  Batch:
    src = masked input ids, tgt_out = original ids at MLM positions (pad
    elsewhere); tgt_in is unused.  V need not be a multiple of 8 (BERT's
    30522): the logits rows are then laid out with a padded pitch.
    """

    def _mask_sites(self, s_src, enc_seed, s_tgt, dec_seed, ts: int, tt: int):
        d, f = self.cfg.d_model, self.cfg.d_ff
        slot = lambda t: t.storage_offset()      # noqa: E731
        sites = [(slot(s_src), ts * d, "src")]
        for i in range(self.cfg.n_enc):
            g = f"enc{i}"
            sites += [(slot(enc_seed.site(i, 0)), ts * d, g), (slot(enc_seed.site(i, 1)), ts * f, g),
                      (slot(enc_seed.site(i, 2)), ts * d, g)]
        return sites

    def register_seeds(self, seeds: SeedTable, seed: int, step: int, p_drop: float):
        cfg = self.cfg
        seeds.reset()
        seeds.set_step(step)
        s_src = seeds.slot(derive_seed(seed, step, 0))
        enc_seed = _LayerSeed(seeds, derive_seed(seed, step, 1))
        if p_drop > 0.0:
            for i in range(cfg.n_enc):
                for k in range(3):
                    enc_seed.site(i, k)
        return s_src, enc_seed, None, None

    def _forward_backward(self, params, batch: Batch, *, p_drop, alpha, seed, step, arena, sink,
                          compute_grads, grad_scale, trace, strategy, capture, validate,
                          upload_seeds) -> ModelOutput:
        cfg = self.cfg
        ctx = _lib.context()
        arena = arena or NullArena(ctx.device)
        stash = ActivationStash()
        sink = GradSink() if sink is None else sink
        if isinstance(sink, _ViewSink):
            sink.arena = arena
        if validate:
            validate_batch(batch, cfg)
        src = K.dev(batch.src, torch.int64)
        tgt_out = K.dev(batch.tgt_out, torch.int64).reshape(-1)
        src_len = K.dev(batch.src_len, torch.int64)
        b, ls = src.shape
        d, n, v = cfg.d_model, cfg.n_heads, cfg.vocab
        params = {k: (t if isinstance(t, torch.Tensor) else K.dev(t)) for k, t in params.items()}
        dt = self.act_dtype(params)
        sdt = _stat_dtype(dt)
        emb_cfg = EmbeddingConfig(scale=cfg.scale, vocab=v, max_len=cfg.max_len,
                                  learned_positional=cfg.learned_positional)
        tok_emb = _as_dt(params["tok_emb"], dt)
        pos = _as_dt(self._positional(params, dt), dt)
        enc_mask = AttentionMask("padding", src_len)
        seeds = self.seed_table(ctx.device)
        s_src, enc_seed, _, _ = self.register_seeds(seeds, seed, step, p_drop)
        if p_drop > 0.0 and upload_seeds:
            seeds.upload()
        bank = _MASKS
        if bank is not None and p_drop > 0.0 and dt != torch.float64:
            bank.prepare(lambda ts, tt: self._mask_sites(s_src, enc_seed, None, None, ts, tt),
                         b * ls, b * ls, K._drop_args(p_drop)[1])
            bank.generate(seeds.dev, stamp=bank.stamp, want=seeds.step_slot())
            bank.active = True
            arena = _BankArena(arena, bank)

        # --- forward: embedding, encoder stack, final LayerNorm ---
        h = arena.alloc((b, ls, d), dt)
        keep_src = _bank_bits(s_src, b * ls * d) if p_drop > 0.0 else None
        banked = keep_src is not None
        if not banked:
            keep_src = arena.alloc((_nbits(b * ls * d),), torch.uint8)
        K.embedding_forward(tok_emb, pos, src, emb_cfg, p_drop, s_src, out=h, bits_out=keep_src,
                            validate=False,
                            mask=DropoutMask(p=p_drop, bits=keep_src, shape=(b, ls, d)) if banked
                            else None)
        stash.push("src_keep", keep_src)
        enc_w = [EncoderLayerWeights.from_params(params, f"enc{i}.") for i in range(cfg.n_enc)]
        chain = CHAIN_FUSE and cfg.n_enc > 0
        pre = None
        for i in range(cfg.n_enc):
            if chain:
                nxt = (enc_w[i + 1].ln1_w, enc_w[i + 1].ln1_b) if i + 1 < cfg.n_enc else \
                    (params["enc_ln.w"], params["enc_ln.b"])
                h, pre = _enc_fwd_chain(h, enc_w[i], enc_mask, p_drop, enc_seed, n, cfg.eps, arena,
                                        stash, f"enc{i}.", i, pre=pre, next_ln=(*nxt, cfg.eps))
            else:
                h, _ = encoder_layer_forward(h, enc_w[i], enc_mask, p_drop, enc_seed, n_heads=n,
                                             eps=cfg.eps, arena=arena, stash=stash, prefix=f"enc{i}.",
                                             site=i)
        stash.push("enc_ln_in", h)
        if chain:
            enc_out, mu_e, sg_e = pre
        else:
            mu_e, sg_e = arena.alloc((b * ls,), sdt), arena.alloc((b * ls,), sdt)
            enc_out = arena.alloc((b, ls, d), dt)
            K.layernorm_forward(h, _as_dt(params["enc_ln.w"], dt), _as_dt(params["enc_ln.b"], dt),
                                cfg.eps, out=enc_out, mu_out=mu_e, sigma_out=sg_e,
                                check_degenerate=False)

        # --- MLM criterion over every position (pad targets are skipped) ---
        rt = b * ls
        ld = (v + 7) // 8 * 8 if dt in (torch.float16, torch.bfloat16) else v
        logits_buf = arena.alloc((rt, ld), dt)
        logits = logits_buf[:, :v] if ld != v else logits_buf
        # V % 8 != 0 (BERT's 30522): an N = V GEMM has only 2-element alignment and
        # cuBLAS falls back to an sm80 CUTLASS kernel 6x slower than the aligned
        # one; the 8-aligned N = V - V % 8 columns and the few tail columns run as
        # two GEMMs instead
        va = v - v % 8 if ld != v else v
        K.gemm(enc_out.view(rt, d), tok_emb[:va], trans_b=True, out=logits_buf[:, :va])
        if va != v:
            K.gemm(enc_out.view(rt, d), tok_emb[va:], trans_b=True, out=logits_buf[:, va:v])
        row_stats = arena.alloc((2 * rt,), torch.float64)
        out3 = torch.empty(3, dtype=torch.float64, device=ctx.device)
        if dt == torch.float64:
            self._criterion_f64(logits, tgt_out, out3, alpha, batch.pad_id, grad_scale,
                                compute_grads, None)
        else:
            _lib.call("ls2_criterion_fused_ld", logits_buf.data_ptr(), ld, tgt_out.data_ptr(),
                      logits_buf.data_ptr() if compute_grads else None, row_stats.data_ptr(),
                      out3.data_ptr(), None, rt, v, float(alpha), int(batch.pad_id), 1,
                      float(grad_scale), _lib.dtype_code(logits_buf), _lib.stream_handle())
        arena.free(row_stats)
        if isinstance(sink, _ViewSink):
            sink.totals = out3
        out = ModelOutput(out3)
        if not compute_grads:
            stash.drain(arena)
            arena.free(mu_e); arena.free(sg_e)
            arena.free(enc_out)
            arena.free(logits_buf)
            return out

        # --- backward ---
        main_arena = arena
        lane, arena, join = _open_lane(sink, arena, dt)
        denc = arena.alloc((b, ls, d), dt)
        K.gemm(logits_buf[:, :va], tok_emb[:va], out=denc.view(rt, d))   # K-split as above
        if va != v:
            K.gemm(logits_buf[:, va:v], tok_emb[va:], accumulate_into=denc.view(rt, d))
        _wgrad(sink, "tok_emb", logits, enc_out.view(rt, d))
        arena.free(logits_buf); arena.free(enc_out)
        h_in = stash.pop("enc_ln_in")
        dh = arena.alloc((b, ls, d), dt)
        df = None
        if chain:      # fused with the last encoder layer's FFN-tail backward
            ne = cfg.n_enc
            df = _ln_bwd_chain(sink, "", "enc_ln", denc, h_in, params["enc_ln.w"], mu_e, sg_e, dh,
                               None, stash, (f"enc{ne - 1}.", f"enc{ne - 1}."), p_drop, arena)
        else:
            _ln_bwd(sink, "", "enc_ln", denc, h_in, params["enc_ln.w"], mu_e, sg_e, dh, None)
        arena.free(denc); arena.free(mu_e); arena.free(sg_e); arena.free(h_in)
        join()
        _ready(sink, "enc_ln.")
        for i in reversed(range(cfg.n_enc)):
            tp = (f"enc{i - 1}.", f"enc{i - 1}.") if (chain and i > 0) else None
            res = encoder_layer_backward(dh, enc_w[i], stash, sink, n_heads=n, p_drop=p_drop,
                                         arena=arena, prefix=f"enc{i}.", param_prefix=f"enc{i}.",
                                         df_in=df, tail_prev=tp)
            dh, df = res if tp is not None else (res, None)
            join()
            _ready(sink, f"enc{i}.")
        keep_src = stash.pop("src_keep")
        self._embedding_grads(sink, dh, src, keep_src, p_drop, emb_cfg)
        arena.free(dh); arena.free(keep_src)
        join()
        _close_lane(sink, lane)
        _ready(sink, None)
        arena = main_arena
        if len(stash):
            raise ShapeMismatch(f"activation stash leaked {len(stash)} entries")
        for buf in getattr(sink, "deferred_buffers", lambda: [])():
            arena.free(buf)
        return out


def make_model(cfg: ModelConfig):
    """The model class for cfg.arch."""
    return EncoderMLM(cfg) if cfg.arch == "encoder" else Transformer(cfg)
