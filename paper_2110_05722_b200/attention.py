"""Fused attention core used by the layer composition (libls2 ls2_attention_*).

Given the per-(b, h) addressing of include/ls2.h, the layer code passes slices
of the fused projection buffers directly:

  self-attention  Q/K/V = qkv[..., 0:d | d:2d | 2d:3d]   (row stride 3d)
  cross-attention Q = qc (stride d); K_i/V_i = kv_buf slices (stride 2*n_dec*d)

so the contractions, the masked softmax and the head split/merge are one
kernel forward and one kernel backward.  Two kernel families sit behind it:

  * L <= 64 (every T-base / WMT bucket): the tcgen05/TMEM/TMA kernels of
    csrc/attention_tc.cu.  The forward saves per-row softmax statistics
    (float32 [B, H, Lq, 2]) instead of the probabilities and the backward
    recomputes P from them, so the saved state is `alloc_state`'s f32 tensor;
  * 64 < L <= 128: the mma.sync kernels of csrc/attention.cu, which save the
    fp16 probabilities [B, H, Lq, Lk].

Shapes neither covers (non-fp16, head dim != 64, L > 128, dense masks) use the
reference-shaped cuBLAS + softmax-kernel path in model.py.
LS2_FUSED_ATTENTION=0 disables both, LS2_ATTN_TC=0 only the tcgen05 family.
"""

from __future__ import annotations

import os

import torch

from . import _lib
from .kernels import AttentionMask, dev

ENABLED = os.environ.get("LS2_FUSED_ATTENTION", "1") != "0"


def _mask_ok(mask) -> bool:
    return mask is None or (isinstance(mask, AttentionMask) and
                            mask.kind in ("none", "causal", "padding"))


def is_flash(lq: int, lk: int) -> bool:
    """Rows past 128: the flash kernels (self-attention only, see tc_ok)."""
    return max(lq, lk) > 128


def fused_ok(dtype, lq: int, lk: int, hd: int, mask, flash: bool = False) -> bool:
    """A fused kernel takes this attention.  flash=True (self-attention call sites,
    which can hand the backward the forward's output) admits 128 < L <= 512."""
    if not ENABLED or dtype != torch.float16 or not _mask_ok(mask):
        return False
    _lib.load_library()
    if _lib._lib.ls2_attention_supported(lq, lk, hd, _lib.F16):
        return True
    return flash and is_flash(lq, lk) and tc_ok(dtype, lq, lk, hd, mask, flash=True)


def tc_ok(dtype, lq: int, lk: int, hd: int, mask, flash: bool = False) -> bool:
    """The tcgen05 family takes this shape (implies fused_ok)."""
    if not ENABLED or dtype != torch.float16 or not _mask_ok(mask):
        return False
    if mask is not None and mask.kind == "causal" and lq != lk:
        return False
    if is_flash(lq, lk) and not flash:
        return False
    _lib.load_library()
    return bool(_lib._lib.ls2_attention_tc_supported(lq, lk, hd, _lib.F16))


def bias_rows(batch: int, lq: int, lk: int) -> int:
    """Rows of the projection-bias partials the backward leaves: one per batch,
    or one per (batch, 128-row block) for the flash kernels."""
    return batch * ((lq + 127) // 128) if is_flash(lq, lk) else batch


def alloc_state(arena, dtype, batch, heads, lq, lk, hd, mask, flash: bool = False):
    """The forward's saved softmax state for the fused kernels: f32 row
    statistics [B, H, Lq, 2] (tcgen05 family; [.., 4] with room for
    D = rowsum(dO * O) for the flash kernels) or fp16 probabilities
    [B, H, Lq, Lk] (mma.sync family)."""
    if tc_ok(dtype, lq, lk, hd, mask, flash=flash):
        return arena.alloc((batch, heads, lq, 4 if is_flash(lq, lk) else 2), torch.float32)
    return arena.alloc((batch, heads, lq, lk), dtype)


def _mask_args(mask):
    if mask is None or mask.kind == "none":
        return _lib.MASK_NONE, None
    if mask.kind == "causal":
        return _lib.MASK_CAUSAL, None
    return _lib.MASK_PADDING, dev(mask.valid_lens, torch.int64)


def forward(q, ldq, k, ldk, v, ldv, probs, o, ldo, batch, heads, lq, lk, hd, mask, scale):
    """probs: the state from alloc_state (f32 statistics or fp16 probabilities)."""
    kind, lens = _mask_args(mask)
    if probs.dtype == torch.float32:
        # the backward recomputes P, so it needs the same mask: keep it (and the
        # device lens it reads) on the saved state
        probs._ls2_amask = (kind, lens)
        _lib.call("ls2_attention_tc_fwd", q.data_ptr(), ldq, k.data_ptr(), ldk, v.data_ptr(),
                  ldv, probs.data_ptr(), o.data_ptr(), ldo, batch, heads, lq, lk, hd, kind,
                  _lib.ptr(lens), float(scale), _lib.stream_handle())
        return
    _lib.call("ls2_attention_fwd", q.data_ptr(), ldq, k.data_ptr(), ldk, v.data_ptr(), ldv,
              probs.data_ptr(), o.data_ptr(), ldo, batch, heads, lq, lk, hd, kind,
              _lib.ptr(lens), float(scale), _lib.stream_handle())


def backward(q, ldq, k, ldk, v, ldv, probs, dout, lddo, dq, lddq, dk, lddk, dv, lddv, batch,
             heads, lq, lk, hd, scale, colsums=None, o=None, ldo=0):
    """colsums: optional ((buf, col0, ld) or None) x 3 for dQ, dK, dV — f64 rows of
    per-batch (flash: per (batch, 128-row block), see bias_rows) column sums (the
    projection biases' gradient partials).  o: the forward's output (required by
    the flash kernels)."""
    cs = []
    for c in (colsums or (None, None, None)):
        if c is None:
            cs += [None, 0]
        else:
            buf, col0, ld = c
            cs += [buf.data_ptr() + 8 * col0, ld]
    if probs.dtype == torch.float32 and probs.shape[-1] == 4:
        if o is None:
            raise ValueError("the flash attention backward needs the forward output o")
        kind, lens = probs._ls2_amask
        _lib.call("ls2_attention_tc_bwd_o", q.data_ptr(), ldq, k.data_ptr(), ldk, v.data_ptr(),
                  ldv, o.data_ptr(), ldo, probs.data_ptr(), dout.data_ptr(), lddo, dq.data_ptr(),
                  lddq, dk.data_ptr(), lddk, dv.data_ptr(), lddv, batch, heads, lq, lk, hd, kind,
                  _lib.ptr(lens), float(scale), *cs, _lib.stream_handle())
        return
    if probs.dtype == torch.float32:
        kind, lens = probs._ls2_amask
        _lib.call("ls2_attention_tc_bwd", q.data_ptr(), ldq, k.data_ptr(), ldk, v.data_ptr(),
                  ldv, probs.data_ptr(), dout.data_ptr(), lddo, dq.data_ptr(), lddq,
                  dk.data_ptr(), lddk, dv.data_ptr(), lddv, batch, heads, lq, lk, hd, kind,
                  _lib.ptr(lens), float(scale), *cs, _lib.stream_handle())
        return
    _lib.call("ls2_attention_bwd_bias", q.data_ptr(), ldq, k.data_ptr(), ldk, v.data_ptr(), ldv,
              probs.data_ptr(), dout.data_ptr(), lddo, dq.data_ptr(), lddq, dk.data_ptr(), lddk,
              dv.data_ptr(), lddv, batch, heads, lq, lk, hd, float(scale), *cs,
              _lib.stream_handle())
