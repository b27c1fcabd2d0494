"""Fused forward operators — drop-in for F/kernels.py, executed by libls2 on sm_100a.

Same names, arguments, return values, aliasing and errors as the reference
operator API.  Tensors are torch CUDA tensors (numpy / CPU inputs are moved
to the device).  dtype rule (F/kernels.py:31-36): float64 in -> float64 out,
float16/bfloat16/float32 in -> float32 out, unless an `out` buffer is given,
in which case its dtype is the storage type (fp16 activations on the GPU
training path).  Dropout masks are generated on the device with the
reference's counter RNG and kept as 1-bit masks; `DropoutMask.keep`
materializes the dense 0/1 tensor on demand.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import AllMaskedRow, DegenerateRow, SequenceTooLong, ShapeMismatch, TokenOutOfRange
from .numerics import keep_threshold

ROW_SERIAL = "row_serial"
ROW_PARALLEL_TREE = "row_parallel_tree"
SERIAL_COL_LIMIT = 4096
_autotune_cache: dict[tuple[int, int], str] = {}

_F = (torch.float16, torch.bfloat16, torch.float32)
_IO_OK = {(torch.float16, torch.float16), (torch.float16, torch.float32),
          (torch.bfloat16, torch.bfloat16), (torch.bfloat16, torch.float32),
          (torch.float32, torch.float32), (torch.float32, torch.float16),
          (torch.float32, torch.bfloat16), (torch.float64, torch.float64)}


# ---------------------------------------------------------------------------
# tensor plumbing
# ---------------------------------------------------------------------------

def dev(x, dtype=None) -> torch.Tensor:
    """Move/convert an array-like to a contiguous CUDA tensor."""
    ctx = _lib.context()
    if isinstance(x, torch.Tensor):
        t = x
        if t.device != ctx.device:
            t = t.to(ctx.device)
    else:
        a = np.asarray(x)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(ctx.device)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def compute_dtype(*arrays) -> torch.dtype:
    """float64 if any input is float64, else float32 (F/kernels.py:31-36)."""
    for a in arrays:
        if a is None:
            continue
        dt = a.dtype if isinstance(a, torch.Tensor) else np.asarray(a).dtype
        if dt in (torch.float64, np.float64):
            return torch.float64
    return torch.float32


def _tin_for(inputs, tout: torch.dtype) -> torch.dtype:
    dts = {t.dtype for t in inputs if t is not None}
    tin = dts.pop() if len(dts) == 1 else (torch.float64 if torch.float64 in dts else torch.float32)
    if (tin, tout) in _IO_OK:
        return tin
    return torch.float64 if tout == torch.float64 else torch.float32


def io_tensors(inputs, tout):
    """Convert inputs to one dtype the kernels support for output dtype tout."""
    ts = [None if x is None else dev(x) for x in inputs]
    tin = _tin_for(ts, tout)
    return [None if t is None else (t if t.dtype == tin else t.to(tin)).contiguous() for t in ts], tin


def _out(out, shape, dtype, device):
    if out is None:
        return torch.empty(shape, dtype=dtype, device=device), None
    if tuple(out.shape) != tuple(shape) and out.numel() != int(np.prod(shape)):
        raise ShapeMismatch(f"out has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if out.is_contiguous():
        return out, None
    tmp = torch.empty(shape, dtype=out.dtype, device=out.device)
    return tmp, out          # copy back after the kernel


def _finish(res, orig):
    if orig is not None:
        orig.copy_(res.view(orig.shape))
        return orig
    return res


def host_tokens(tokens) -> np.ndarray | None:
    if isinstance(tokens, torch.Tensor):
        return tokens.detach().cpu().numpy() if tokens.device.type == "cpu" else None
    return np.asarray(tokens)


# ---------------------------------------------------------------------------
# reduction strategy (F/kernels.py:80-106)
# ---------------------------------------------------------------------------

_STRATEGY_CODE = {None: 0, ROW_SERIAL: 1, ROW_PARALLEL_TREE: 2}


def _strategy_code(strategy) -> int:
    """`strategy=` of the softmax family -> LS2_SOFTMAX_* (None: the shape rule).
    Any other value reduces serially, as the reference's _reduce_rows does
    (F/kernels.py:73-77)."""
    return _STRATEGY_CODE.get(strategy, 1)


def select_softmax_strategy(rows: int, cols: int, autotune: bool = False) -> str:
    """Shape -> strategy.  On the GPU the two strategies are the register-cached
    sub-warp template (row_serial) and the CTA-per-row template
    (row_parallel_tree); autotune times both once per shape and caches the winner."""
    if rows < 1 or cols < 1:
        raise ShapeMismatch(f"bad softmax shape ({rows}, {cols})")
    key = (rows, cols)
    if key in _autotune_cache:
        return _autotune_cache[key]
    if not autotune:
        return ROW_SERIAL if cols <= SERIAL_COL_LIMIT else ROW_PARALLEL_TREE
    probe = torch.sin(torch.arange(rows * cols, dtype=torch.float32, device=_lib.context().device)
                      ).reshape(rows, cols)
    out = torch.empty_like(probe)
    timings = {}
    for strat in (ROW_SERIAL, ROW_PARALLEL_TREE):
        softmax_forward(probe, out=out, strategy=strat)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        softmax_forward(probe, out=out, strategy=strat)
        torch.cuda.synchronize()
        timings[strat] = time.perf_counter() - t0
    _autotune_cache[key] = min(timings, key=timings.get)
    return _autotune_cache[key]


# ---------------------------------------------------------------------------
# masks and caches
# ---------------------------------------------------------------------------

@dataclass
class AttentionMask:
    """Which key positions each query may attend to (F/kernels.py:113-136).

    kind: "none", "causal" or "padding" (valid_lens = per-sequence prefix).
    The kernels evaluate the mask from indices; keep_array() materializes it.
    """

    kind: str = "none"
    valid_lens: object = None

    def keep_array(self, lq: int, lk: int):
        if self.kind == "none":
            return None
        ctx = _lib.context()
        if self.kind == "causal":
            return torch.ones((lq, lk), dtype=torch.bool, device=ctx.device).tril()
        if self.kind == "padding":
            lens = self.lens_host()
            if lens.min() < 1 or lens.max() > lk:
                raise ShapeMismatch("padding valid length outside [1, Lk]")
            lt = torch.as_tensor(lens, device=ctx.device)
            return (torch.arange(lk, device=ctx.device)[None, :] < lt[:, None])[:, None, None, :]
        raise ShapeMismatch(f"unknown mask kind {self.kind!r}")

    def lens_host(self) -> np.ndarray:
        v = self.valid_lens
        return v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v)


class DropoutMask:
    """Per-element keep indicator plus drop probability (F/kernels.py:147-152).

    Stored densely (`keep`) or as the device bit mask the kernels produce
    (`bits`: byte i>>3, bit i&7 of the flat index).  Either view is derived
    from the other on demand.
    """

    def __init__(self, keep=None, p: float = 0.0, bits: torch.Tensor | None = None,
                 shape: tuple | None = None, dense_dtype: torch.dtype = torch.float32):
        if keep is not None and not isinstance(keep, torch.Tensor):
            keep = dev(keep)
        self._keep = keep
        self.p = p
        self.bits = bits
        self.shape = tuple(keep.shape) if (shape is None and keep is not None) else shape
        self.dense_dtype = dense_dtype

    @property
    def keep(self) -> torch.Tensor:
        if self._keep is None and self.p == 0.0 and self.shape is not None:
            self._keep = torch.ones(self.shape, dtype=self.dense_dtype,
                                    device=_lib.context().device)
        elif self._keep is None and self.bits is not None:
            t = torch.empty(self.shape, dtype=self.dense_dtype, device=self.bits.device)
            _lib.call("ls2_bits_to_dense", self.bits.data_ptr(), t.data_ptr(),
                      _lib.dtype_code(t), self.numel, _lib.stream_handle())
            self._keep = t
        return self._keep

    @keep.setter
    def keep(self, v):
        self._keep = v

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 0

    def bitmask(self) -> torch.Tensor:
        if self.bits is None:
            k = self._keep.contiguous()
            b = torch.empty((self.numel + 7) // 8, dtype=torch.uint8, device=k.device)
            _lib.call("ls2_dense_to_bits", k.data_ptr(), _lib.dtype_code(k), b.data_ptr(),
                      self.numel, _lib.stream_handle())
            self.bits = b
        return self.bits


def _drop_args(p: float):
    if not 0.0 <= p < 1.0:
        raise ShapeMismatch(f"dropout probability {p} outside [0, 1)")
    if p == 0.0:
        return 0, 0, 1.0
    return 1, keep_threshold(p), 1.0 / (1.0 - p)


def _seed_args(seed):
    """(value, device pointer) for a dropout seed given as an int or as a
    1-element uint64/int64 CUDA tensor (graph-replayable per-step seeds)."""
    if isinstance(seed, torch.Tensor):
        return 0, seed.data_ptr()
    return int(seed) & ((1 << 64) - 1), None


def _new_bits(n: int, device) -> torch.Tensor:
    return torch.empty((n + 7) // 8, dtype=torch.uint8, device=device)


def make_dropout_mask(shape, p: float, seed: int, dtype=torch.float32, out=None) -> DropoutMask:
    """Counter-RNG dropout mask: element i kept iff rand(seed, i) >= p."""
    use, thresh, _ = _drop_args(p)
    shape = tuple(int(s) for s in shape)
    ctx = _lib.context()
    n = int(np.prod(shape))
    dtype = _torch_dtype(dtype)
    keep = out if out is not None else torch.empty(shape, dtype=dtype, device=ctx.device)
    if not use:
        keep.fill_(1)
        return DropoutMask(keep=keep, p=p, shape=shape)
    bits = _new_bits(n, ctx.device)
    _lib.call("ls2_dropout_bits", bits.data_ptr(), n, seed & ((1 << 64) - 1), None, thresh,
              _lib.stream_handle())
    _lib.call("ls2_bits_to_dense", bits.data_ptr(), keep.data_ptr(), _lib.dtype_code(keep), n,
              _lib.stream_handle())
    return DropoutMask(keep=keep, p=p, bits=bits, shape=shape)


def _torch_dtype(dt):
    if isinstance(dt, torch.dtype):
        return dt
    return {np.dtype(np.float16): torch.float16, np.dtype(np.float32): torch.float32,
            np.dtype(np.float64): torch.float64}[np.dtype(dt)]


@dataclass
class LNCache:
    mu: torch.Tensor
    sigma: torch.Tensor
    xhat: torch.Tensor | None = None


@dataclass
class SoftmaxCache:
    probs: torch.Tensor


@dataclass
class EmbeddingConfig:
    scale: float
    vocab: int
    max_len: int
    learned_positional: bool = True

    def __post_init__(self):
        if self.scale <= 0:
            raise ShapeMismatch(f"embedding scale must be > 0, got {self.scale}")
        if self.vocab < 2:
            raise ShapeMismatch(f"vocab must be >= 2, got {self.vocab}")


# ---------------------------------------------------------------------------
# embedding (F/kernels.py:203-228)
# ---------------------------------------------------------------------------

def check_tokens(tokens, vocab: int, max_len: int | None = None):
    t = host_tokens(tokens)
    if t is not None:
        if t.ndim != 2:
            raise ShapeMismatch(f"tokens must be [B, L], got shape {t.shape}")
        if max_len is not None and t.shape[1] > max_len:
            raise SequenceTooLong(f"sequence length {t.shape[1]} > max_len {max_len}")
        if t.size and (t.min() < 0 or t.max() >= vocab):
            raise TokenOutOfRange(f"token ids outside [0, {vocab})")
        return dev(t.astype(np.int64))
    tk = tokens
    if tk.dim() != 2:
        raise ShapeMismatch(f"tokens must be [B, L], got shape {tuple(tk.shape)}")
    if max_len is not None and tk.shape[1] > max_len:
        raise SequenceTooLong(f"sequence length {tk.shape[1]} > max_len {max_len}")
    tk = dev(tk, torch.int64)
    if tk.numel() and (int(tk.min()) < 0 or int(tk.max()) >= vocab):   # API-level sync
        raise TokenOutOfRange(f"token ids outside [0, {vocab})")
    return tk


def embedding_forward(emb, pos, tokens, cfg: EmbeddingConfig, p_drop: float, seed: int,
                      out=None, keep_out=None, bits_out=None, validate: bool = True,
                      mask: DropoutMask | None = None):
    """y[b,i,:] = keep * (s * emb[tokens[b,i],:] + pos[i,:]) / (1 - p).

    mask: reuse an existing mask's bits instead of drawing them (injected masks).
    Returns ([B, L, d], DropoutMask)."""
    tk = check_tokens(tokens, cfg.vocab, cfg.max_len) if validate else tokens
    b, l = tk.shape
    tout = out.dtype if out is not None else compute_dtype(emb, pos)
    (e, p), tin = io_tensors([emb, pos], tout)
    d = e.shape[1]
    y, orig = _out(out, (b, l, d), tout, e.device)
    use, thresh, ds = _drop_args(p_drop)
    n = b * l * d
    gen = 1
    if mask is not None and use:
        bits, gen = mask.bitmask(), 0
    else:
        bits = bits_out if bits_out is not None else (_new_bits(n, e.device) if use else None)
    _lib.call("ls2_embedding_fwd", e.data_ptr(), p.data_ptr(), tk.data_ptr(), y.data_ptr(),
              _lib.ptr(bits), None, b, l, d, cfg.vocab, float(cfg.scale), use, gen,
              *_seed_args(seed), thresh, ds, _lib.dtype_code(tin), _lib.dtype_code(tout),
              _lib.stream_handle())
    y = _finish(y, orig)
    if mask is None or not use:
        mask = DropoutMask(p=p_drop, bits=bits, shape=(b, l, d), dense_dtype=tout)
    if keep_out is not None:
        _fill_keep(keep_out, mask)
        mask.keep = keep_out
    return y, mask


def _fill_keep(keep_out, mask: DropoutMask):
    if mask.bits is None:
        keep_out.fill_(1)
    else:
        _lib.call("ls2_bits_to_dense", mask.bits.data_ptr(), keep_out.data_ptr(),
                  _lib.dtype_code(keep_out), mask.numel, _lib.stream_handle())


# ---------------------------------------------------------------------------
# LayerNorm (F/kernels.py:235-270)
# ---------------------------------------------------------------------------

def layernorm_forward(x, w, b, eps: float = 1e-5, out=None, mu_out=None, sigma_out=None,
                      check_degenerate: bool = True):
    """Normalize each row of x[..., m]; returns (y, LNCache(mu, sigma))."""
    xs = x.shape if isinstance(x, torch.Tensor) else np.asarray(x).shape
    m = xs[-1]
    if m < 2:
        raise ShapeMismatch(f"layernorm needs m >= 2, got {m}")
    tout = out.dtype if out is not None else compute_dtype(x, w, b)
    (xt, wt, bt), tin = io_tensors([x, w, b], tout)
    r = xt.numel() // m
    y, orig = _out(out, xt.shape, tout, xt.device)
    tstat = torch.float64 if tin == torch.float64 else torch.float32
    if mu_out is not None and mu_out.dtype in (torch.float32, torch.float64) and mu_out.is_contiguous():
        tstat = mu_out.dtype
    mu = mu_out if (mu_out is not None and mu_out.dtype == tstat and mu_out.is_contiguous()) else \
        torch.empty(r, dtype=tstat, device=xt.device)
    sg = sigma_out if (sigma_out is not None and sigma_out.dtype == tstat and sigma_out.is_contiguous()) else \
        torch.empty(r, dtype=tstat, device=xt.device)
    flag = None
    if eps == 0.0 and check_degenerate:
        flag = torch.zeros(1, dtype=torch.int32, device=xt.device)
    _lib.call("ls2_layernorm_fwd", xt.data_ptr(), wt.data_ptr(), bt.data_ptr(), y.data_ptr(),
              mu.data_ptr(), sg.data_ptr(), _lib.ptr(flag), r, m, float(eps),
              _lib.dtype_code(tin), _lib.dtype_code(tout), _lib.dtype_code(tstat),
              _lib.stream_handle())
    if flag is not None and int(flag.item()):
        raise DegenerateRow("zero-variance row with eps = 0")
    if mu_out is not None and mu is not mu_out:
        mu_out.copy_(mu.view(mu_out.shape))
        mu = mu_out
    if sigma_out is not None and sg is not sigma_out:
        sigma_out.copy_(sg.view(sigma_out.shape))
        sg = sigma_out
    return _finish(y, orig), LNCache(mu=mu, sigma=sg)


# ---------------------------------------------------------------------------
# softmax family (F/kernels.py:277-331)
# ---------------------------------------------------------------------------

def mask_spec(mask, shape):
    """(kind, lq, heads, lens tensor, dense uint8 keep) for the kernel."""
    c = shape[-1]
    lq = shape[-2] if len(shape) >= 2 else 1
    if mask is None:
        return _lib.MASK_NONE, 1, 1, None, None
    if isinstance(mask, AttentionMask):
        if mask.kind == "none":
            return _lib.MASK_NONE, 1, 1, None, None
        if mask.kind == "causal":
            return _lib.MASK_CAUSAL, lq, 1, None, None
        if mask.kind == "padding":
            lens = mask.lens_host() if not isinstance(mask.valid_lens, torch.Tensor) else None
            if lens is not None and (lens.min() < 1 or lens.max() > c):
                raise ShapeMismatch("padding valid length outside [1, Lk]")
            lt = dev(mask.valid_lens, torch.int64)
            if len(shape) != 4:
                raise ShapeMismatch("padding masks apply to [B, N, Lq, Lk] scores")
            return _lib.MASK_PADDING, lq, shape[1], lt, None
        raise ShapeMismatch(f"unknown mask kind {mask.kind!r}")
    keep = dev(mask, torch.bool)
    keep = torch.broadcast_to(keep, tuple(shape)).to(torch.uint8).contiguous()
    if not bool(keep.reshape(-1, c).any(dim=1).all()):
        raise AllMaskedRow("softmax row with every position masked")
    return _lib.MASK_DENSE, lq, 1, None, keep


def softmax_forward(x, mask=None, out=None, strategy: str | None = None, in_scale: float = 1.0):
    """Row softmax over the last axis with an optional attention mask.

    Masked positions are excluded from max and sum and emit exactly 0;
    returns (y, SoftmaxCache(probs=y)); out may alias x.  in_scale folds the
    attention 1/sqrt(hd) into the same pass (F/model.py:368)."""
    tout = out.dtype if out is not None else compute_dtype(x)
    (xt,), tin = io_tensors([x], tout)
    shape = tuple(xt.shape)
    c = shape[-1]
    r = xt.numel() // c
    kind, lq, heads, lens, dense = mask_spec(mask, shape)
    y, orig = _out(out, shape, tout, xt.device)
    _lib.call("ls2_softmax_fwd_strategy", xt.data_ptr(), y.data_ptr(), r, c, kind, lq, heads,
              _lib.ptr(lens), _lib.ptr(dense), float(in_scale), None, _strategy_code(strategy),
              _lib.dtype_code(tin), _lib.dtype_code(tout), _lib.stream_handle())
    y = _finish(y, orig)
    return y, SoftmaxCache(probs=y)


def log_softmax_forward(h, out=None, strategy: str | None = None):
    """logq_i = (h_i - max) - log Z; never forms q and takes its log."""
    tout = out.dtype if out is not None else compute_dtype(h)
    (ht,), tin = io_tensors([h], tout)
    c = ht.shape[-1]
    if c < 2:
        raise ShapeMismatch(f"log_softmax needs >= 2 classes, got {c}")
    y, orig = _out(out, ht.shape, tout, ht.device)
    _lib.call("ls2_log_softmax_fwd_strategy", ht.data_ptr(), y.data_ptr(), ht.numel() // c, c,
              _strategy_code(strategy), _lib.dtype_code(tin), _lib.dtype_code(tout),
              _lib.stream_handle())
    return _finish(y, orig)


# ---------------------------------------------------------------------------
# label-smoothed cross entropy (F/kernels.py:338-360)
# ---------------------------------------------------------------------------

def _targets(targets, rows: int):
    t = dev(targets, torch.int64).reshape(-1)
    if t.numel() != rows:
        raise ShapeMismatch(f"{t.numel()} targets for {rows} rows")
    return t


def ls_cross_entropy_forward(logq, targets, alpha: float, pad_id: int | None = None):
    """(loss_sum, token_count) of smoothed CE over non-pad tokens."""
    (lq,), tin = io_tensors([logq], compute_dtype(logq))
    v = lq.shape[-1]
    r = lq.numel() // v
    t = _targets(targets, r)
    ctx = _lib.context()
    stats = torch.empty(2 * max(r, 1), dtype=torch.float64, device=lq.device)
    out3 = torch.zeros(3, dtype=torch.float64, device=lq.device)
    bad = torch.zeros(1, dtype=torch.int32, device=lq.device)
    _lib.call("ls2_ls_ce_fwd", lq.data_ptr(), t.data_ptr(), stats.data_ptr(), out3.data_ptr(),
              bad.data_ptr(), r, v, float(alpha), 0 if pad_id is None else int(pad_id),
              0 if pad_id is None else 1, _lib.dtype_code(tin), _lib.stream_handle())
    o = out3.cpu().numpy()
    if int(bad.item()):
        raise TokenOutOfRange(f"target outside [0, {v})")
    del ctx
    return float(o[0]), int(o[1])


# ---------------------------------------------------------------------------
# fused element-wise tails (F/kernels.py:367-403)
# ---------------------------------------------------------------------------

def bias_dropout_residual(x, bias, residual, p: float, seed: int, out=None, keep_out=None,
                          bits_out=None, mask: DropoutMask | None = None):
    """y = keep * (x + bias) / (1 - p) + residual; returns (y, DropoutMask).

    mask: reuse an existing mask's bits instead of generating (injected masks)."""
    tout = out.dtype if out is not None else compute_dtype(x, bias, residual)
    (xt, bt, rt), tin = io_tensors([x, bias, residual], tout)
    shape = tuple(xt.shape)
    cols = shape[-1]
    n = xt.numel()
    if rt.numel() != n or bt.numel() != cols:
        raise ShapeMismatch("bias_dropout_residual operand shapes disagree")
    y, orig = _out(out, shape, tout, xt.device)
    use, thresh, ds = _drop_args(p)
    gen = 1
    if mask is not None and use:
        bits, gen = mask.bitmask(), 0
    else:
        bits = bits_out if bits_out is not None else (_new_bits(n, xt.device) if use else None)
    _lib.call("ls2_bias_dropout_residual_fwd", xt.data_ptr(), bt.data_ptr(), rt.data_ptr(),
              y.data_ptr(), _lib.ptr(bits), n // cols, cols, use, gen, *_seed_args(seed),
              thresh, ds, _lib.dtype_code(tin), _lib.dtype_code(tout), _lib.stream_handle())
    y = _finish(y, orig)
    dm = mask if (mask is not None and use) else DropoutMask(p=p, bits=bits, shape=shape,
                                                             dense_dtype=tout)
    if keep_out is not None:
        _fill_keep(keep_out, dm)
        dm.keep = keep_out
    return y, dm


def bias_relu_dropout(x, bias, p: float, seed: int, out=None, keep_out=None, relu_out=None,
                      bits_out=None, relu_bits_out=None, mask: DropoutMask | None = None):
    """y = keep * relu(x + bias) / (1 - p); returns (y, DropoutMask, relu_mask).

    relu_mask records strict positivity of (x + bias).  With relu_bits_out the
    relu mask is returned as a DropoutMask-style bit container (model path)."""
    tout = out.dtype if out is not None else compute_dtype(x, bias)
    (xt, bt), tin = io_tensors([x, bias], tout)
    shape = tuple(xt.shape)
    cols = shape[-1]
    n = xt.numel()
    if bt.numel() != cols:
        raise ShapeMismatch("bias_relu_dropout bias length != last dim")
    y, orig = _out(out, shape, tout, xt.device)
    use, thresh, ds = _drop_args(p)
    gen = 1
    if mask is not None and use:
        bits, gen = mask.bitmask(), 0
    else:
        bits = bits_out if bits_out is not None else (_new_bits(n, xt.device) if use else None)
    rbits = relu_bits_out if relu_bits_out is not None else _new_bits(n, xt.device)
    _lib.call("ls2_bias_relu_dropout_fwd", xt.data_ptr(), bt.data_ptr(), y.data_ptr(),
              _lib.ptr(bits), rbits.data_ptr(), n // cols, cols, use, gen,
              *_seed_args(seed), thresh, ds, _lib.dtype_code(tin), _lib.dtype_code(tout),
              _lib.stream_handle())
    y = _finish(y, orig)
    dm = mask if (mask is not None and use) else DropoutMask(p=p, bits=bits, shape=shape,
                                                             dense_dtype=tout)
    if keep_out is not None:
        _fill_keep(keep_out, dm)
        dm.keep = keep_out
    relu = ReluMask(bits=rbits, shape=shape, dense_dtype=tout)
    if relu_out is not None:
        _lib.call("ls2_bits_to_dense", rbits.data_ptr(), relu_out.data_ptr(),
                  _lib.dtype_code(relu_out), n, _lib.stream_handle())
        return y, dm, relu_out
    if relu_bits_out is not None:
        return y, dm, relu
    return y, dm, relu.dense()


@dataclass
class ReluMask:
    """Bit container for the relu mask (same layout as DropoutMask bits)."""

    bits: torch.Tensor
    shape: tuple
    dense_dtype: torch.dtype = torch.float32

    def dense(self) -> torch.Tensor:
        t = torch.empty(self.shape, dtype=self.dense_dtype, device=self.bits.device)
        _lib.call("ls2_bits_to_dense", self.bits.data_ptr(), t.data_ptr(), _lib.dtype_code(t),
                  int(np.prod(self.shape)), _lib.stream_handle())
        return t


def as_bits(mask, shape) -> torch.Tensor:
    """Bit view of a relu/dropout mask given densely or as bits."""
    if isinstance(mask, (DropoutMask, ReluMask)):
        if isinstance(mask, DropoutMask):
            return mask.bitmask()
        return mask.bits
    return DropoutMask(keep=dev(mask), p=0.5, shape=tuple(shape)).bitmask()


# ---------------------------------------------------------------------------
# GEMM (F/kernels.py:413-447) on cuBLAS
# ---------------------------------------------------------------------------

GEMM_BLOCK_K = 512


def _mat_layout(t: torch.Tensor):
    """(transposed?, ld) for the last two dims of t, or None if not a matrix view."""
    r, c = t.shape[-2], t.shape[-1]
    sr, sc = t.stride(-2), t.stride(-1)
    if sc == 1 and (sr >= max(c, 1) or r == 1):
        return False, max(sr, c)
    if sr == 1 and (sc >= max(r, 1) or c == 1):
        return True, max(sc, r)
    return None


def _joint_levels(views):
    """Batch levels shared by all operands: [(count, [stride per operand])] x 2,
    merging adjacent batch dims wherever every operand allows it; None if more
    than two levels remain."""
    shape = list(views[0].shape[:-2])
    dims = [(shape[i], [v.stride()[i] for v in views]) for i in range(len(shape)) if shape[i] != 1]
    i = 0
    while i + 1 < len(dims):
        (n0, s0), (n1, s1) = dims[i], dims[i + 1]
        if all(a == n1 * b for a, b in zip(s0, s1)):
            dims[i:i + 2] = [(n0 * n1, s1)]
        else:
            i += 1
    if len(dims) > 2:
        return None
    while len(dims) < 2:
        dims.insert(0, (1, [0] * len(views)))
    return dims


def gemm_list(a_list, b_list, outs, trans_a: bool = False, trans_b: bool = False,
              alpha: float = 1.0, beta: float = 0.0):
    """outs[i] = alpha * op(a_list[i]) @ op(b_list[i]) + beta * outs[i] for products
    of ONE shape and layout at unrelated addresses, as cuBLAS pointer-array
    batches of up to 64 (ls2_gemm_list).  Contiguous 2-D CUDA operands only."""
    ctx = _lib.context()
    if not (len(a_list) == len(b_list) == len(outs)) or not a_list:
        raise ShapeMismatch("gemm_list: operand lists differ in length or are empty")
    a0, b0, c0 = a_list[0], b_list[0], outs[0]
    for group in (a_list, b_list, outs):
        for t in group:
            if t.dim() != 2 or not t.is_contiguous() or not t.is_cuda:
                raise ShapeMismatch("gemm_list: contiguous 2-D CUDA operands only")
            if t.shape != group[0].shape or t.dtype != group[0].dtype:
                raise ShapeMismatch("gemm_list: every product must have one shape and dtype")
    if a0.dtype != b0.dtype:
        raise ShapeMismatch("gemm_list: A and B dtypes differ")
    m, k = (a0.shape[1], a0.shape[0]) if trans_a else tuple(a0.shape)
    kb, n = (b0.shape[1], b0.shape[0]) if trans_b else tuple(b0.shape)
    if k != kb or tuple(c0.shape) != (m, n):
        raise ShapeMismatch(f"gemm_list: op(A) {m}x{k}, op(B) {kb}x{n}, C {tuple(c0.shape)}")
    for lo in range(0, len(a_list), 64):
        A, B, C = a_list[lo:lo + 64], b_list[lo:lo + 64], outs[lo:lo + 64]
        cnt = len(A)
        key = ("list",) + tuple(t.data_ptr() for t in A + B + C)
        # the table is filled by the first call (the eager first step of a bucket,
        # before its graph is captured) and reused: planned-arena addresses are static
        scratch = ctx.ptr_cache.get(key)
        ready = 1
        if scratch is None:
            scratch = torch.empty(3 * cnt, dtype=torch.int64, device=ctx.device)
            ctx.ptr_cache[key] = scratch
            ready = 0
        arr = ctypes.c_void_p * cnt
        _lib.call("ls2_gemm_list", ctx.blas_handle(), int(trans_a), int(trans_b), m, n, k,
                  float(alpha), arr(*[t.data_ptr() for t in A]), a0.shape[1],
                  arr(*[t.data_ptr() for t in B]), b0.shape[1], float(beta),
                  arr(*[t.data_ptr() for t in C]), n, cnt, _lib.dtype_code(a0),
                  _lib.dtype_code(c0), scratch.data_ptr(), ready, _lib.stream_handle())
    return outs


def gemm(a, b, trans_a: bool = False, trans_b: bool = False, accumulate_into=None, out=None,
         alpha: float = 1.0, beta: float | None = None):
    """C = alpha * op(a) @ op(b) (+ accumulate_into); fp32 (fp64 for f64) accumulation.

    Stacked operands with identical leading dims are multiplied slice-wise as
    one cuBLAS batch (strided, or pointer-array for two-level head views)."""
    ctx = _lib.context()
    A = a.to(ctx.device) if isinstance(a, torch.Tensor) else dev(a)
    B = b.to(ctx.device) if isinstance(b, torch.Tensor) else dev(b)
    cdt = compute_dtype(A, B)
    if A.dtype != B.dtype or A.dtype not in (torch.float16, torch.bfloat16, torch.float32,
                                             torch.float64):
        A, B = A.to(cdt), B.to(cdt)
    av = A.transpose(-1, -2) if trans_a else A
    bv = B.transpose(-1, -2) if trans_b else B
    if av.shape[-1] != bv.shape[-2]:
        raise ShapeMismatch(f"inner dims {av.shape[-1]} != {bv.shape[-2]}")
    if av.shape[:-2] != bv.shape[:-2]:
        raise ShapeMismatch(f"batch dims {tuple(av.shape[:-2])} != {tuple(bv.shape[:-2])}")
    m, k, n = av.shape[-2], av.shape[-1], bv.shape[-1]
    oshape = tuple(av.shape[:-2]) + (m, n)
    if accumulate_into is not None:
        C, beta_v = accumulate_into, 1.0 if beta is None else beta
    elif out is not None:
        C, beta_v = out, 0.0 if beta is None else beta
    else:
        C = torch.empty(oshape, dtype=cdt, device=ctx.device)
        beta_v = 0.0
    tc = C.dtype
    if (A.dtype == torch.float64) != (tc == torch.float64):
        A, B = A.to(tc if tc == torch.float64 else torch.float32), B.to(tc if tc == torch.float64 else torch.float32)
    elif tc not in (A.dtype, torch.float32):
        A, B = A.to(torch.float32), B.to(torch.float32)
    av = A.transpose(-1, -2) if trans_a else A
    bv = B.transpose(-1, -2) if trans_b else B
    Cv = C.view(oshape) if tuple(C.shape) != oshape else C
    la, lb, lc = _mat_layout(av), _mat_layout(bv), _mat_layout(Cv)
    tmp_c = None
    if lc is None or lc[0]:
        tmp_c = torch.empty(oshape, dtype=tc, device=ctx.device)
        if beta_v != 0.0:
            tmp_c.copy_(Cv)
    Cw = Cv if tmp_c is None else tmp_c
    lv = _joint_levels([av, bv, Cw]) if (la is not None and lb is not None) else None
    if lv is None:
        av = av.contiguous() if la is None or True else av
        bv = bv.contiguous()
        if tmp_c is None and not Cw.is_contiguous():
            tmp_c = Cw.contiguous()
            Cw = tmp_c
        la, lb, lc = _mat_layout(av), _mat_layout(bv), _mat_layout(Cw)
        lv = _joint_levels([av, bv, Cw])
    lc = _mat_layout(Cw)
    (n1, s1), (n2, s2) = lv
    scratch, ready = None, 0
    collapsible = n1 == 1 or n2 == 1 or all(a == n2 * b for a, b in zip(s1, s2))
    if not collapsible:
        # pointer-array batch: arrays cached per (addresses, strides) -> filled once;
        # the planned arena makes the addresses static, so graph replays reuse them
        key = (av.data_ptr(), bv.data_ptr(), Cw.data_ptr(), tuple(s1), tuple(s2), n1, n2,
               av.element_size(), Cw.element_size())
        scratch = ctx.ptr_cache.get(key)
        if scratch is None:
            scratch = torch.empty(3 * n1 * n2, dtype=torch.int64, device=ctx.device)
            ctx.ptr_cache[key] = scratch
        else:
            ready = 1
    _lib.call("ls2_gemm", ctx.blas_handle(), int(la[0]), int(lb[0]), m, n, k, float(alpha),
              av.data_ptr(), la[1], s1[0], s2[0], bv.data_ptr(), lb[1], s1[1], s2[1],
              float(beta_v), Cw.data_ptr(), lc[1], s1[2], s2[2], n1, n2,
              _lib.dtype_code(av), _lib.dtype_code(tc), _lib.ptr(scratch), ready,
              _lib.stream_handle())
    if tmp_c is not None:
        Cv.copy_(tmp_c)
    return C
