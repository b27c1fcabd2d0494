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


class _Alloc:
    def alloc(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device="cuda")


CASES = [(64, 8, 64, 64, "padding"), (64, 8, 64, 64, "causal"), (3, 2, 37, 37, "causal"),
         (4, 16, 128, 128, "padding"), (5, 3, 20, 52, "padding"), (2, 4, 7, 100, "none"),
         (2, 2, 128, 16, "none"), (113, 8, 36, 36, "padding"), (10, 8, 48, 48, "causal"),
         (7, 2, 33, 45, "padding"),
         # tcgen05 packing: G = 64 // max(Lq, Lk) sequences per tile, ragged last
         # group, odd tile counts, cross-attention with Lq != Lk
         (512, 8, 8, 8, "padding"), (341, 8, 12, 12, "causal"), (3, 2, 5, 5, "none"),
         (33, 4, 16, 24, "padding"), (5, 3, 64, 64, "none"), (9, 1, 30, 31, "padding"),
         (17, 8, 60, 60, "causal"), (1, 1, 1, 1, "none"),
         # 64 < L <= 128: one 128-row tcgen05 tile per (batch, head)
         (64, 16, 128, 128, "causal"), (6, 4, 65, 65, "padding"), (5, 2, 100, 77, "padding"),
         (3, 3, 90, 128, "none"), (16, 12, 128, 128, "padding")]


@pytest.mark.parametrize("impl", ["tc", "mma"])
@pytest.mark.parametrize("B,NH,Lq,Lk,kind", CASES)
def test_fused_attention_vs_oracle(B, NH, Lq, Lk, kind, impl):
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
    assert ATT.fused_ok(torch.float16, Lq, Lk, 64, mask)
    if impl == "tc":
        if not ATT.tc_ok(torch.float16, Lq, Lk, 64, mask):
            assert kind == "causal" and Lq != Lk
            pytest.skip("causal cross-attention (Lq != Lk) stays on the mma.sync family")
        probs = ATT.alloc_state(_Alloc(), torch.float16, B, NH, Lq, Lk, 64, mask)
        assert probs.dtype == torch.float32 and probs.shape == (B, NH, Lq, 2)
    else:
        probs = torch.empty((B, NH, Lq, Lk), dtype=torch.float16, device="cuda")
    o = torch.empty((B, Lq, d), dtype=torch.float16, device="cuda")
    scale = 1.0 / math.sqrt(64)
    ATT.forward(q, d, k, 2 * d, v, 2 * d, probs, o, d, B, NH, Lq, Lk, 64, mask, scale)
    dq = torch.empty_like(q)
    dkv = torch.zeros((B, Lk, 2 * d), dtype=torch.float16, device="cuda")
    dout = torch.tensor(dod, device="cuda")
    cs = torch.full((B, 3 * d), float("nan"), dtype=torch.float64, device="cuda")
    ATT.backward(q, d, k, 2 * d, v, 2 * d, probs, dout, d, dq, d, dkv[..., :d], 2 * d,
                 dkv[..., d:], 2 * d, B, NH, Lq, Lk, 64, scale,
                 colsums=((cs, 0, 3 * d), (cs, d, 3 * d), (cs, 2 * d, 3 * d)))
    hs = lambda x, L: x.astype(np.float32).reshape(B, L, NH, 64).transpose(0, 2, 1, 3)  # noqa
    p, oo, dqq, dkk, dvv = _ref(hs(qd, Lq), hs(kd, Lk), hs(vd, Lk), keep, hs(dod, Lq), scale)
    merge = lambda x: x.transpose(0, 2, 1, 3).reshape(B, x.shape[2], d)  # noqa
    if impl == "mma":
        assert np.abs(H(probs).astype(np.float32) - p).max() <= 2e-3
        if keep is not None:
            assert np.all(H(probs)[~np.broadcast_to(keep, p.shape)] == 0)
    else:
        # stats = (max of the scaled unmasked scores in the log2 domain, i.e. times
        # log2(e), and 1 / sum exp(s - max)) per row
        s = np.einsum("bhqd,bhkd->bhqk", hs(qd, Lq), hs(kd, Lk)) * np.float32(scale)
        if keep is not None:
            s = np.where(np.broadcast_to(keep, s.shape), s, -np.inf)
        m = s.max(-1)
        iz = 1.0 / np.exp(s - m[..., None]).sum(-1)
        st = H(probs)
        m2 = m * np.float32(1.4426950408889634)
        assert np.abs(st[..., 0] - m2).max() <= 1e-2 * max(1.0, np.abs(m2).max())
        assert np.abs(st[..., 1] - iz).max() <= 1e-2 * np.abs(iz).max()
    for got, want in ((H(o), merge(oo)), (H(dq), merge(dqq)), (H(dkv[..., :d]), merge(dkk)),
                      (H(dkv[..., d:]), merge(dvv))):
        got = got.astype(np.float32)
        assert np.abs(got - want).max() <= 2e-2 * max(1.0, np.abs(want).max())
    # bias-gradient partials: column sums of the stored fp16 dQ / dK / dV.  The
    # mma.sync family leaves one row per batch; the tcgen05 family one row per
    # packed group of G sequences (at the group's first batch, zeros in the
    # others).  Either way the B rows sum to the bias gradient.
    want_cs = np.concatenate([H(dq).astype(np.float64).sum(1), H(dkv).astype(np.float64).sum(1)],
                             axis=1)
    got_cs = H(cs)
    assert np.isfinite(got_cs).all()
    tol = 1e-3 * max(1.0, np.abs(want_cs).sum(0).max())
    assert np.abs(got_cs.sum(0) - want_cs.sum(0)).max() <= tol
    if impl == "mma":
        assert np.abs(got_cs - want_cs).max() <= 1e-3 * max(1.0, np.abs(want_cs).max())
    else:
        G = max(1, 64 // max(Lq, Lk))      # L > 64: one 128-row tile per (b, h)
        grp = np.add.reduceat(want_cs, np.arange(0, B, G), axis=0)
        assert np.abs(got_cs[::G] - grp).max() <= 1e-3 * max(1.0, np.abs(grp).max())
        assert np.all(np.delete(got_cs, np.arange(0, B, G), axis=0) == 0)


@pytest.mark.parametrize("B,NH,L,kind", [(64, 8, 64, "padding"), (512, 8, 8, "causal"),
                                         (64, 16, 128, "causal"), (16, 12, 128, "padding"),
                                         (113, 8, 36, "padding"), (341, 8, 12, "none")])
def test_tc_attention_matches_mma_kernels(B, NH, L, kind):
    """The tcgen05 and mma.sync families on the same inputs: outputs and
    gradients agree to fp16 rounding (both accumulate in fp32)."""
    rng = np.random.default_rng(7 + L)
    d = 64 * NH
    qkv = torch.tensor((rng.normal(size=(B, L, 3 * d)) * 0.8).astype(np.float16), device="cuda")
    dout = torch.tensor(rng.normal(size=(B, L, d)).astype(np.float16), device="cuda")
    lens = torch.tensor(rng.integers(1, L + 1, B), device="cuda")
    mask = AttentionMask(kind, lens) if kind == "padding" else AttentionMask(kind)
    q, k, v = qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]
    outs = {}
    for impl in ("tc", "mma"):
        st = ATT.alloc_state(_Alloc(), torch.float16, B, NH, L, L, 64, mask) if impl == "tc" \
            else torch.empty((B, NH, L, L), dtype=torch.float16, device="cuda")
        o = torch.empty((B, L, d), dtype=torch.float16, device="cuda")
        ATT.forward(q, 3 * d, k, 3 * d, v, 3 * d, st, o, d, B, NH, L, L, 64, mask, 0.125)
        dqkv = torch.empty_like(qkv)
        ATT.backward(q, 3 * d, k, 3 * d, v, 3 * d, st, dout, d, dqkv[..., :d], 3 * d,
                     dqkv[..., d:2 * d], 3 * d, dqkv[..., 2 * d:], 3 * d, B, NH, L, L, 64, 0.125)
        outs[impl] = (H(o).astype(np.float32), H(dqkv).astype(np.float32))
    for a, b in zip(outs["tc"], outs["mma"]):
        assert np.abs(a - b).max() <= 1e-2 * max(1.0, np.abs(b).max())


def test_fused_attention_gates():
    assert not ATT.fused_ok(torch.float32, 64, 64, 64, None)
    assert not ATT.fused_ok(torch.float16, 64, 200, 64, None)
    assert not ATT.fused_ok(torch.float16, 64, 64, 32, None)
    assert not ATT.fused_ok(torch.float16, 64, 64, 64, torch.ones(64, 64, dtype=torch.bool))


@pytest.mark.parametrize("B,NH,L,kind", [(4, 4, 512, "padding"), (3, 2, 256, "none"),
                                         (2, 3, 200, "causal"), (5, 2, 129, "padding"),
                                         (2, 12, 384, "padding"), (16, 12, 512, "padding")])
def test_flash_attention_vs_oracle(B, NH, L, kind):
    """128 < L <= 512 self-attention (BERT-512): the flash kernels (128-row blocks,
    K / V streamed, scores never in HBM; backward = dQ pass + dK/dV pass with
    D = rowsum(dO * O)) against the f32 oracle, and the bias partials (one row per
    (batch, 128-row block)) against the column sums of the stored gradients."""
    rng = np.random.default_rng(B * 1000 + L)
    d = 64 * NH
    qkv_h = (rng.normal(size=(B, L, 3 * d)) * 0.8).astype(np.float16)
    qkv_h[..., 2 * d:] = rng.normal(size=(B, L, d)).astype(np.float16)
    dod = rng.normal(size=(B, L, d)).astype(np.float16)
    lens = rng.integers(1, L + 1, B)
    lens[0] = L
    mask = AttentionMask(kind, torch.tensor(lens, device="cuda")) if kind == "padding" else \
        AttentionMask(kind)
    keep = {"padding": O.pad_keep(lens, L, L), "causal": O.causal_keep(L, L), "none": None}[kind]
    assert ATT.fused_ok(torch.float16, L, L, 64, mask, flash=True)
    assert not ATT.fused_ok(torch.float16, L, L, 64, mask)          # cross-attention sites
    qkv = torch.tensor(qkv_h, device="cuda")
    q, k, v = qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]
    st = ATT.alloc_state(_Alloc(), torch.float16, B, NH, L, L, 64, mask, flash=True)
    assert st.dtype == torch.float32 and st.shape == (B, NH, L, 4)
    o = torch.empty((B, L, d), dtype=torch.float16, device="cuda")
    scale = 1.0 / math.sqrt(64)
    ATT.forward(q, 3 * d, k, 3 * d, v, 3 * d, st, o, d, B, NH, L, L, 64, mask, scale)
    dqkv = torch.empty_like(qkv)
    nrow = ATT.bias_rows(B, L, L)
    assert nrow == B * ((L + 127) // 128)
    cs = torch.full((nrow, 3 * d), float("nan"), dtype=torch.float64, device="cuda")
    dout = torch.tensor(dod, device="cuda")
    ATT.backward(q, 3 * d, k, 3 * d, v, 3 * d, st, dout, d, dqkv[..., :d], 3 * d,
                 dqkv[..., d:2 * d], 3 * d, dqkv[..., 2 * d:], 3 * d, B, NH, L, L, 64, scale,
                 colsums=((cs, 0, 3 * d), (cs, d, 3 * d), (cs, 2 * d, 3 * d)), o=o, ldo=d)
    hs = lambda x: x.astype(np.float32).reshape(B, L, NH, 64).transpose(0, 2, 1, 3)  # noqa
    merge = lambda x: x.transpose(0, 2, 1, 3).reshape(B, L, d)  # noqa
    _, oo, dqq, dkk, dvv = _ref(hs(qkv_h[..., :d]), hs(qkv_h[..., d:2 * d]),
                                hs(qkv_h[..., 2 * d:]), keep, hs(dod), scale)
    got_dqkv = H(dqkv).astype(np.float32)
    for got, want in ((H(o).astype(np.float32), merge(oo)), (got_dqkv[..., :d], merge(dqq)),
                      (got_dqkv[..., d:2 * d], merge(dkk)), (got_dqkv[..., 2 * d:], merge(dvv))):
        assert np.abs(got - want).max() <= 2e-2 * max(1.0, np.abs(want).max())
        assert np.linalg.norm(got - want) <= 1e-2 * max(1e-6, np.linalg.norm(want))
    got_cs = H(cs)
    assert np.isfinite(got_cs).all()
    want_cs = H(dqkv).astype(np.float64).sum(1)                     # [B, 3d]
    per_b = got_cs.reshape(B, -1, 3 * d).sum(1)
    assert np.abs(per_b - want_cs).max() <= 1e-3 * max(1.0, np.abs(want_cs).max())
