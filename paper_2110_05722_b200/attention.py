"""Fused attention core used by the layer composition (libls2 ls2_attention_*).

Given the per-(b, h) addressing of include/ls2.h, the layer code passes slices
of the fused projection buffers directly:

  self-attention  Q/K/V = qkv[..., 0:d | d:2d | 2d:3d]   (row stride 3d)
  cross-attention Q = qc (stride d); K_i/V_i = kv_buf slices (stride 2*n_dec*d)

so the contractions, the masked softmax and the head split/merge are one
kernel forward and one kernel backward.  Shapes it does not cover (non-fp16,
head dim != 64, L > 128, dense masks) use the reference-shaped cuBLAS +
softmax-kernel path in model.py.  LS2_FUSED_ATTENTION=0 disables it.
"""

from __future__ import annotations

import os

import torch

from . import _lib
from .kernels import AttentionMask, dev

ENABLED = os.environ.get("LS2_FUSED_ATTENTION", "1") != "0"


def fused_ok(dtype, lq: int, lk: int, hd: int, mask) -> bool:
    if not ENABLED or dtype != torch.float16:
        return False
    if mask is not None and not (isinstance(mask, AttentionMask) and
                                 mask.kind in ("none", "causal", "padding")):
        return False
    _lib.load_library()
    return bool(_lib._lib.ls2_attention_supported(lq, lk, hd, _lib.F16))


def _mask_args(mask):
    if mask is None or mask.kind == "none":
        return _lib.MASK_NONE, None
    if mask.kind == "causal":
        return _lib.MASK_CAUSAL, None
    return _lib.MASK_PADDING, dev(mask.valid_lens, torch.int64)


def forward(q, ldq, k, ldk, v, ldv, probs, o, ldo, batch, heads, lq, lk, hd, mask, scale):
    kind, lens = _mask_args(mask)
    _lib.call("ls2_attention_fwd", q.data_ptr(), ldq, k.data_ptr(), ldk, v.data_ptr(), ldv,
              probs.data_ptr(), o.data_ptr(), ldo, batch, heads, lq, lk, hd, kind,
              _lib.ptr(lens), float(scale), _lib.stream_handle())


def backward(q, ldq, k, ldk, v, ldv, probs, dout, lddo, dq, lddq, dk, lddk, dv, lddv, batch,
             heads, lq, lk, hd, scale, colsums=None):
    """colsums: optional ((buf, col0, ld) or None) x 3 for dQ, dK, dV — f64 rows of
    per-batch column sums (the projection biases' gradient partials)."""
    cs = []
    for c in (colsums or (None, None, None)):
        if c is None:
            cs += [None, 0]
        else:
            buf, col0, ld = c
            cs += [buf.data_ptr() + 8 * col0, ld]
    _lib.call("ls2_attention_bwd_bias", q.data_ptr(), ldq, k.data_ptr(), ldk, v.data_ptr(), ldv,
              probs.data_ptr(), dout.data_ptr(), lddo, dq.data_ptr(), lddq, dk.data_ptr(), lddk,
              dv.data_ptr(), lddv, batch, heads, lq, lk, hd, float(scale), *cs,
              _lib.stream_handle())
