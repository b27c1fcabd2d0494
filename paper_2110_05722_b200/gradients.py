"""Analytic backward operators — drop-in for F/gradients.py, executed by libls2.

Parameter-gradient reductions (bias, LayerNorm weight/bias, positional table)
are deterministic two-stage column sums; only the token-table scatter uses
atomics, as in LightSeq2.  The extra keyword arguments (`dbias_out`,
`dw_out`/`db_out`, `beta`, `dres`, `out_scale`) let the model write parameter
gradients straight into the fp32 gradient workspace and fuse the residual add
and the attention 1/sqrt(hd) into the same pass.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatch, TargetOutOfRange
from .kernels import (DropoutMask, EmbeddingConfig, LNCache, SoftmaxCache, _out, _finish,
                      _targets, as_bits, check_tokens, compute_dtype, dev, io_tensors)


def _scratch(name, nbytes):
    return _lib.context().scratch(name, nbytes)


def embedding_backward(dy, tokens, mask: DropoutMask, cfg: EmbeddingConfig, dE_out=None,
                       dP_out=None, beta_pos: int = 0, validate: bool = True):
    """dE[w] = s * sum_{tokens == w} keep * dy / (1 - p); dP[l] = sum_b keep*dy/(1-p).

    Rows of tokens that never occur stay exactly zero (F/gradients.py:20-44).
    With dE_out/dP_out the gradients accumulate into caller buffers (fp32/fp64)."""
    tk = check_tokens(tokens, cfg.vocab) if validate else tokens
    gdt = torch.float64 if compute_dtype(dy) == torch.float64 else torch.float32
    (d_,), tin = io_tensors([dy], gdt)
    if tuple(d_.shape[:2]) != tuple(tk.shape):
        raise ShapeMismatch(f"dy {tuple(d_.shape)} does not cover tokens {tuple(tk.shape)}")
    b, l, d = d_.shape
    de = dE_out if dE_out is not None else torch.zeros((cfg.vocab, d), dtype=gdt, device=d_.device)
    dp = None
    if cfg.learned_positional:
        dp = dP_out if dP_out is not None else torch.empty((cfg.max_len, d), dtype=gdt,
                                                           device=d_.device)
    use = 1 if mask.p > 0.0 else 0
    bits = mask.bitmask() if use else None
    _lib.call("ls2_embedding_bwd", d_.data_ptr(), tk.data_ptr(), _lib.ptr(bits), de.data_ptr(),
              _lib.ptr(dp), _lib.dtype_code(de), int(beta_pos), b, l, d, cfg.max_len,
              float(cfg.scale), use, 1.0 / (1.0 - mask.p) if use else 1.0, _lib.dtype_code(tin),
              _lib.stream_handle())
    return de, dp


def ls_cross_entropy_backward(probs, targets, alpha: float, pad_id: int | None = None,
                              grad_scale: float = 1.0, out=None, check: bool = True):
    """dh_i = q_i - a/V - (1 - a)[i == truth]; pad rows emit zero; x grad_scale."""
    tout = out.dtype if out is not None else compute_dtype(probs)
    (pr,), tin = io_tensors([probs], tout)
    v = pr.shape[-1]
    r = pr.numel() // v
    t = _targets(targets, r)
    dh, orig = _out(out, pr.shape, tout, pr.device)
    bad = torch.zeros(1, dtype=torch.int32, device=pr.device) if check else None
    _lib.call("ls2_ls_ce_bwd", pr.data_ptr(), t.data_ptr(), dh.data_ptr(), _lib.ptr(bad), r, v,
              float(alpha), 0 if pad_id is None else int(pad_id), 0 if pad_id is None else 1,
              float(grad_scale), _lib.dtype_code(tin), _lib.dtype_code(tout), _lib.stream_handle())
    if bad is not None and int(bad.item()):
        raise TargetOutOfRange(f"target outside [0, {v})")
    return _finish(dh, orig)


def softmax_backward(dy, cache: SoftmaxCache, out=None, out_scale: float = 1.0):
    """dx_i = q_i * (dy_i - sum_j dy_j q_j) (x out_scale); out may alias dy."""
    q = cache.probs
    dys = dy.shape if isinstance(dy, torch.Tensor) else tuple(dev(dy).shape)
    if tuple(dys) != tuple(q.shape):
        raise ShapeMismatch(f"dy {tuple(dys)} != probs {tuple(q.shape)}")
    tout = out.dtype if out is not None else compute_dtype(dy, q)
    (d_, qq), tin = io_tensors([dy, q], tout)
    c = d_.shape[-1]
    dx, orig = _out(out, d_.shape, tout, d_.device)
    _lib.call("ls2_softmax_bwd", d_.data_ptr(), qq.data_ptr(), dx.data_ptr(), d_.numel() // c, c,
              float(out_scale), _lib.dtype_code(tin), _lib.dtype_code(tout), _lib.stream_handle())
    return _finish(dx, orig)


def layernorm_backward(dy, x, w, cache: LNCache, out=None, dres=None, dw_out=None, db_out=None,
                       beta: int = 0, partials_out=None):
    """Rearranged LayerNorm backward: dx plus affine parameter grads (dw, db).

    dres (optional) is added to dx in the same pass (the residual branch of
    F/model.py:468,508)."""
    tout = out.dtype if out is not None else compute_dtype(dy, x, w)
    (d_, xt, wt, rt), tin = io_tensors([dy, x, w, dres], tout)
    if d_.shape != xt.shape:
        raise ShapeMismatch(f"dy {tuple(d_.shape)} != x {tuple(xt.shape)}")
    m = xt.shape[-1]
    r = xt.numel() // m
    pdt = compute_dtype(dy, x, w)
    # host (numpy) statistics keep their precision: f64 stats stay f64
    mu, sg = (v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v))
              for v in (cache.mu, cache.sigma))
    tstat = mu.dtype if mu.dtype in (torch.float32, torch.float64) else torch.float32
    mu = dev(mu, tstat).reshape(-1)
    sg = dev(sg, tstat).reshape(-1)
    dx, orig = _out(out, xt.shape, tout, xt.device)
    if partials_out is not None:      # deferred finish: partial[blk][2][m] stays in partials_out
        dw = db = None
        ws = partials_out
    else:
        dw = dw_out if dw_out is not None else torch.empty(m, dtype=pdt, device=xt.device)
        db = db_out if db_out is not None else torch.empty(m, dtype=pdt, device=xt.device)
        if dw.dtype != db.dtype:
            raise ShapeMismatch("dw/db dtypes differ")
        ws = _scratch("reduce", _lib.call_i64("ls2_layernorm_bwd_ws_bytes", r, m))
    _lib.call("ls2_layernorm_bwd", d_.data_ptr(), xt.data_ptr(), wt.data_ptr(), mu.data_ptr(),
              sg.data_ptr(), _lib.ptr(rt), dx.data_ptr(), _lib.ptr(dw), _lib.ptr(db),
              _lib.dtype_code(dw if dw is not None else pdt), int(beta), ws.data_ptr(), r, m,
              _lib.dtype_code(tin), _lib.dtype_code(tout), _lib.dtype_code(tstat),
              _lib.stream_handle())
    return _finish(dx, orig), dw, db


def bias_dropout_residual_backward(dy, mask: DropoutMask, out=None, dbias_out=None,
                                   beta: int = 0, partials_out=None):
    """dx = keep * dy / (1 - p); dbias = column sums of dx; dresidual IS dy.

    partials_out: leave dbias as per-block partial sums there (deferred finish);
    dbias is then returned as None."""
    tout = out.dtype if out is not None else compute_dtype(dy)
    (d_,), tin = io_tensors([dy], tout)
    cols = d_.shape[-1]
    rows = d_.numel() // cols
    dx, orig = _out(out, d_.shape, tout, d_.device)
    pdt = compute_dtype(dy)
    if partials_out is not None:
        db, ws = None, partials_out
    else:
        db = dbias_out if dbias_out is not None else torch.empty(cols, dtype=pdt, device=d_.device)
        ws = _scratch("reduce", _lib.call_i64("ls2_colsum_ws_bytes", rows, cols))
    use = 1 if mask.p > 0.0 else 0
    bits = mask.bitmask() if use else None
    _lib.call("ls2_bias_dropout_residual_bwd", d_.data_ptr(), _lib.ptr(bits), dx.data_ptr(),
              _lib.ptr(db), _lib.dtype_code(db if db is not None else pdt), int(beta),
              ws.data_ptr(), rows, cols, use, 1.0 / (1.0 - mask.p) if use else 1.0,
              _lib.dtype_code(tin), _lib.dtype_code(tout), _lib.stream_handle())
    return _finish(dx, orig), db, dy


def bias_relu_dropout_backward(dy, dropmask: DropoutMask, relu_mask, out=None, dbias_out=None,
                               beta: int = 0, partials_out=None):
    """dx = relu_mask * keep * dy / (1 - p); dbias reduces dx over rows.

    partials_out: deferred finish, as in bias_dropout_residual_backward."""
    tout = out.dtype if out is not None else compute_dtype(dy)
    (d_,), tin = io_tensors([dy], tout)
    cols = d_.shape[-1]
    rows = d_.numel() // cols
    dx, orig = _out(out, d_.shape, tout, d_.device)
    pdt = compute_dtype(dy)
    if partials_out is not None:
        db, ws = None, partials_out
    else:
        db = dbias_out if dbias_out is not None else torch.empty(cols, dtype=pdt, device=d_.device)
        ws = _scratch("reduce", _lib.call_i64("ls2_colsum_ws_bytes", rows, cols))
    use = 1 if dropmask.p > 0.0 else 0
    kb = dropmask.bitmask() if use else None
    rb = as_bits(relu_mask, d_.shape)
    _lib.call("ls2_bias_relu_dropout_bwd", d_.data_ptr(), _lib.ptr(kb), rb.data_ptr(),
              dx.data_ptr(), _lib.ptr(db), _lib.dtype_code(db if db is not None else pdt),
              int(beta), ws.data_ptr(), rows, cols, use, 1.0 / (1.0 - dropmask.p) if use else 1.0,
              _lib.dtype_code(tin), _lib.dtype_code(tout), _lib.stream_handle())
    return _finish(dx, orig), db


def column_sum(x, out=None, beta: int = 0, partials_out=None):
    """Deterministic float64-accumulated column sums of x[..., c] (bias grads).
    partials_out: leave per-block partials there (deferred finish), return None."""
    xt = x if isinstance(x, torch.Tensor) else dev(x)
    if not xt.is_contiguous():
        xt = xt.contiguous()
    cols = xt.shape[-1]
    rows = xt.numel() // cols
    if partials_out is not None:
        _lib.call("ls2_colsum", xt.data_ptr(), _lib.dtype_code(xt), None, _lib.F32, 0,
                  partials_out.data_ptr(), rows, cols, _lib.stream_handle())
        return None
    o = out if out is not None else torch.empty(cols, dtype=compute_dtype(xt), device=xt.device)
    ws = _scratch("reduce", _lib.call_i64("ls2_colsum_ws_bytes", rows, cols))
    _lib.call("ls2_colsum", xt.data_ptr(), _lib.dtype_code(xt), o.data_ptr(), _lib.dtype_code(o),
              int(beta), ws.data_ptr(), rows, cols, _lib.stream_handle())
    return o
