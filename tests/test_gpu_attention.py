"""Fused attention kernel (libls2 ls2_attention_fwd/bwd) vs the oracle's unfused
composition (scores -> masked softmax -> PV and the reference backward,
F/model.py:362-376, 482-495).  fp16 storage: 2e-2 relative tolerance."""

import math

import numpy as np
import pytest
import torch

from oracle import lsport as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2110_05722_b200 import attention as ATT
    from paper_2110_05722_b200.kernels import AttentionMask


def H(t):
    return t.detach().cpu().numpy()


def _ref(q, k, v, keep, dout, scale):
    """[B,H,L,64] float32 numpy reference of fwd + bwd."""
    s = np.einsum("bhqd,bhkd->bhqk", q, k) * np.float32(scale)
    p = O.softmax_fwd(s, keep)
    o = np.einsum("bhqk,bhkd->bhqd", p, v)
    dp = np.einsum("bhqd,bhkd->bhqk", dout, v)
    ds = O.softmax_bwd(dp, p) * np.float32(scale)
    return p, o, np.einsum("bhqk,bhkd->bhqd", ds, k), np.einsum("bhqk,bhqd->bhkd", ds, q), \
        np.einsum("bhqk,bhqd->bhkd", p, dout)


@pytest.mark.parametrize("B,NH,Lq,Lk,kind", [(64, 8, 64, 64, "padding"), (64, 8, 64, 64, "causal"),
                                             (3, 2, 37, 37, "causal"), (4, 16, 128, 128, "padding"),
                                             (5, 3, 20, 52, "padding"), (2, 4, 7, 100, "none"),
                                             (2, 2, 128, 16, "none"), (113, 8, 36, 36, "padding"),
                                             (10, 8, 48, 48, "causal"), (7, 2, 33, 45, "padding")])
def test_fused_attention_vs_oracle(B, NH, Lq, Lk, kind):
    rng = np.random.default_rng(B * 100 + Lq)
    d = 64 * NH
    # self-attention style packed [B, L, 3d] for q/k/v when Lq == Lk, separate otherwise
    qd = (rng.normal(size=(B, Lq, d)) * 0.8).astype(np.float16)
    kd = (rng.normal(size=(B, Lk, d)) * 0.8).astype(np.float16)
    vd = rng.normal(size=(B, Lk, d)).astype(np.float16)
    dod = rng.normal(size=(B, Lq, d)).astype(np.float16)
    lens = rng.integers(1, Lk + 1, B)
    lens[0] = Lk
    mask = AttentionMask(kind, torch.tensor(lens, device="cuda")) if kind == "padding" else \
        AttentionMask(kind)
    keep = {"padding": O.pad_keep(lens, Lq, Lk), "causal": O.causal_keep(Lq, Lk), "none": None}[kind]
    kv = torch.tensor(np.concatenate([kd, vd], axis=-1), device="cuda")   # strided K/V views
    q = torch.tensor(qd, device="cuda")
    k, v = kv[..., :d], kv[..., d:]
    probs = torch.empty((B, NH, Lq, Lk), dtype=torch.float16, device="cuda")
    o = torch.empty((B, Lq, d), dtype=torch.float16, device="cuda")
    scale = 1.0 / math.sqrt(64)
    assert ATT.fused_ok(torch.float16, Lq, Lk, 64, mask)
    ATT.forward(q, d, k, 2 * d, v, 2 * d, probs, o, d, B, NH, Lq, Lk, 64, mask, scale)
    dq = torch.empty_like(q)
    dkv = torch.zeros((B, Lk, 2 * d), dtype=torch.float16, device="cuda")
    dout = torch.tensor(dod, device="cuda")
    ATT.backward(q, d, k, 2 * d, v, 2 * d, probs, dout, d, dq, d, dkv[..., :d], 2 * d,
                 dkv[..., d:], 2 * d, B, NH, Lq, Lk, 64, scale)
    hs = lambda x, L: x.astype(np.float32).reshape(B, L, NH, 64).transpose(0, 2, 1, 3)  # noqa
    p, oo, dqq, dkk, dvv = _ref(hs(qd, Lq), hs(kd, Lk), hs(vd, Lk), keep, hs(dod, Lq), scale)
    merge = lambda x: x.transpose(0, 2, 1, 3).reshape(B, x.shape[2], d)  # noqa
    assert np.abs(H(probs).astype(np.float32) - p).max() <= 2e-3
    if keep is not None:
        assert np.all(H(probs)[~np.broadcast_to(keep, p.shape)] == 0)
    for got, want in ((H(o), merge(oo)), (H(dq), merge(dqq)), (H(dkv[..., :d]), merge(dkk)),
                      (H(dkv[..., d:]), merge(dvv))):
        got = got.astype(np.float32)
        assert np.abs(got - want).max() <= 2e-2 * max(1.0, np.abs(want).max())


def test_fused_attention_gates():
    assert not ATT.fused_ok(torch.float32, 64, 64, 64, None)
    assert not ATT.fused_ok(torch.float16, 64, 200, 64, None)
    assert not ATT.fused_ok(torch.float16, 64, 64, 32, None)
    assert not ATT.fused_ok(torch.float16, 64, 64, 64, torch.ones(64, 64, dtype=torch.bool))
