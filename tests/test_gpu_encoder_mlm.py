"""BERT-shaped encoder + tied MLM criterion (BASELINE.json configs[3]) vs the
oracle composition (oracle/lsport.py OracleEncoderMLM, built from the pinned
reference pieces).  f64: 1e-9; f32: 2e-5; fp16 activations: 2e-2 (north star).
V = 43 exercises the padded logits pitch (V % 8 != 0) on the 16-bit path."""

import numpy as np
import pytest
import torch

from oracle import lsport as O

pytestmark = pytest.mark.gpu

from paper_2110_05722_b200 import model as M                 # host-importable (no GPU needed)
from paper_2110_05722_b200.config import RunConfig, TrainConfig
from paper_2110_05722_b200.data import MLMTask

if torch.cuda.is_available():
    from paper_2110_05722_b200.engine import TrainingEngine


def H(t):
    return t.detach().cpu().numpy()


def _cfg(d=16, heads=4, dff=24, vocab=43, max_len=12, n_enc=2):
    return M.ModelConfig(n_enc=n_enc, n_dec=0, d_model=d, n_heads=heads, d_ff=dff, vocab=vocab,
                         max_len=max_len, arch="encoder")


def _batch(cfg, b=3, l=10, seed=5):
    t = MLMTask(b, l, cfg.vocab, seed=seed, mask_prob=0.3).batch(2)
    lens = np.array([l, l - 3, l - 1][:b])
    return M.Batch(t.src, t.tgt_in, t.tgt_out, lens, 0)


def _oracle(cfg, params, batch, p, dt):
    om = O.OracleEncoderMLM(cfg.n_enc, cfg.d_model, cfg.n_heads, cfg.d_ff, cfg.vocab, cfg.max_len)
    P = {k: H(v).astype(dt) for k, v in params.items()}
    return om.forward_backward(P, batch.src, batch.tgt_out, batch.src_len, pad_id=0, p=p,
                               alpha=0.1, seed=11, step=4, grad_scale=1.0)


def test_encoder_param_spec_matches_oracle_layout():
    cfg = _cfg()
    assert [(n, tuple(s)) for n, s in M.param_spec(cfg)] == \
        [(n, tuple(s)) for n, s in O.encoder_param_shapes(2, 16, 24, 43, 12)]


@pytest.mark.parametrize("tag,dt,tol", [("f64", torch.float64, 1e-9), ("f32", torch.float32, 2e-5)])
def test_encoder_mlm_forward_backward_vs_oracle(tag, dt, tol):
    cfg = _cfg()
    m = M.make_model(cfg)
    params = {k: v.to(dt) for k, v in M.init_params(cfg, seed=3).items()}
    batch = _batch(cfg)
    sink = M.GradSink()
    out = m.forward_backward(params, batch, p_drop=0.2, alpha=0.1, seed=11, step=4, sink=sink)
    loss, cnt, correct, G = _oracle(cfg, params, batch, 0.2, np.float64 if tag == "f64" else np.float32)
    assert out.token_count == cnt and out.correct == correct
    assert abs(out.loss_sum - loss) <= tol * abs(loss)
    for name, _ in M.param_spec(cfg):
        ref = G[name]
        got = H(sink.store[name])
        assert np.abs(got - ref).max() <= tol * max(1.0, np.abs(ref).max()), name


@pytest.mark.parametrize("vocab,d,heads,l", [(43, 16, 4, 10), (1003, 128, 2, 64)])
def test_encoder_mlm_fp16_vs_oracle(vocab, d, heads, l):
    """fp16 activations (padded logits pitch for V % 8 != 0; the fused attention
    kernel at head dim 64) vs the f32 oracle on the fp16-rounded parameters."""
    cfg = _cfg(d=d, heads=heads, dff=2 * d, vocab=vocab, max_len=l + 2)
    m = M.make_model(cfg)
    p32 = M.init_params(cfg, seed=3)
    p16 = {k: v.half() for k, v in p32.items()}
    batch = _batch(cfg, b=3, l=l)
    sink = M.GradSink()
    out = m.forward_backward(p16, batch, p_drop=0.1, alpha=0.1, seed=11, step=4, sink=sink)
    loss, cnt, correct, G = _oracle(cfg, {k: v.float() for k, v in p16.items()}, batch, 0.1,
                                    np.float32)
    assert out.token_count == cnt
    assert abs(out.loss_sum - loss) <= 2e-2 * abs(loss)
    # 2e-2 on the loss and the last layers; fp16 activation rounding compounds
    # through the stack, so the first layer's gradients get 4e-2 (d = 16 is the
    # noisiest case: rounding error does not average out over 16 columns)
    for name, tol in (("tok_emb", 2e-2), ("enc1.ffn.w2", 2e-2), ("enc_ln.w", 2e-2),
                      ("enc0.attn.wqkv", 4e-2), ("pos_emb", 4e-2)):
        ref, got = G[name], H(sink.store[name]).astype(np.float32)
        assert np.linalg.norm(got - ref) <= tol * max(np.linalg.norm(ref), 1e-6), name


class _PatternMLM(MLMTask):
    """Learnable MLM data: each row counts up from a random start (mod V), so a
    masked token is predictable from its neighbours."""

    def batch(self, step):
        t = super().batch(step)
        rng = np.random.default_rng(step)
        start = rng.integers(2, self.v, (self.b, 1))
        tok = 2 + (start - 2 + np.arange(self.l)[None, :]) % (self.v - 2)
        mlm = t.tgt_out != self.pad_id
        return M.Batch(np.where(mlm, self.mask_id, tok), np.where(mlm, self.mask_id, tok),
                       np.where(mlm, tok, self.pad_id), t.src_len, self.pad_id)


@pytest.mark.parametrize("force_dp", [False, True])
def test_encoder_mlm_engine_trains(force_dp):
    from paper_2110_05722_b200.dist import DataParallel
    cfg = _cfg(d=128, heads=2, dff=256, vocab=301, max_len=32)
    run = RunConfig(model=cfg, train=TrainConfig(p_drop=0.1, batch_tokens=256, lr=3e-3,
                                                 loss_scale=1.0))
    eng = TrainingEngine(run, task=_PatternMLM(8, 32, 301, seed=1),
                         dp=DataParallel(force=force_dp))
    eng.setup_arena()
    ms = [eng.train_step(s) for s in range(60)]
    assert all(np.isfinite(m.loss) for m in ms) and not ms[-1].skipped
    assert eng._graphs, "bucket graph captured"
    assert np.mean([m.loss for m in ms[-5:]]) < np.mean([m.loss for m in ms[:5]])
