"""Where does the fp16 step's gradient error enter?  (diagnostic, not a test)

Runs two eager T-base engine steps on the GPU (8 x 64 ragged batch of
tests/test_gpu_headline.py), tapping at step 1 the gradient entering each
decoder layer and every cross-attention query gradient (model.GRAD_TAP) and
the ReLU decisions (model.RELU_TAP).  The oracle re-runs step 1 from the
GPU's params in f32 (ReLU decisions injected) and once more with every
stored activation/gradient rounded to fp16 where the GPU stores one (an
"ideal fp16 storage" emulation).  Prints normwise errors of GPU vs f32 and of
the emulation vs f32 at every tap point.

  python tools/diag_parity.py [--steps N] [--json out.json]
"""

import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import lsport as O                                  # noqa: E402
from paper_2110_05722_b200 import model as M                    # noqa: E402
from paper_2110_05722_b200.config import RunConfig, TrainConfig, transformer_base  # noqa: E402
from paper_2110_05722_b200.engine import TrainingEngine         # noqa: E402
from test_gpu_headline import _OneBatch, _ragged_batch, _unpack_bits, _nerr, H  # noqa: E402

r16 = lambda a: O.from_half(O.to_half(a))                       # noqa: E731


class Tapped(O.OracleTransformer):
    """Oracle recording the decoder-backward gradients at the GPU's tap points."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.tap = {}
        self._cross = None

    def dec_bwd(self, dy, c, P, pre, p, G, t):
        i = int(pre[3:-1])
        if i == self.n_dec - 1:
            self.tap[f"dg{self.n_dec}"] = np.array(dy)
        self._cross = pre
        out = super().dec_bwd(dy, c, P, pre, p, G, t)
        self.tap[f"dg{i}"] = np.array(out[0])
        return out

    def _attn_bwd(self, dctxm, pr, q, k, v, t):
        dq, dk, dv = super()._attn_bwd(dctxm, pr, q, k, v, t)
        if self._cross is not None:
            self.tap["dqc:" + self._cross] = np.array(dq)
            self._cross = None
        return dq, dk, dv


def emulate_fp16():
    """Monkeypatch the oracle's elementwise ops to round their outputs to fp16
    and return an oracle class whose GEMM / attention outputs are rounded."""
    orig = {k: getattr(O, k) for k in ["layernorm_fwd", "bias_dropout_residual_fwd",
                                       "bias_relu_dropout_fwd", "embedding_fwd", "layernorm_bwd",
                                       "bias_dropout_residual_bwd", "bias_relu_dropout_bwd"]}
    first = lambda f: (lambda *a, **k: (lambda r: (r16(r[0]),) + tuple(r[1:]))(f(*a, **k)))  # noqa
    O.layernorm_fwd = first(orig["layernorm_fwd"])
    O.bias_dropout_residual_fwd = lambda *a: r16(orig["bias_dropout_residual_fwd"](*a))
    O.bias_relu_dropout_fwd = first(orig["bias_relu_dropout_fwd"])
    O.embedding_fwd = lambda *a: r16(orig["embedding_fwd"](*a))
    O.layernorm_bwd = first(orig["layernorm_bwd"])
    O.bias_dropout_residual_bwd = first(orig["bias_dropout_residual_bwd"])
    O.bias_relu_dropout_bwd = first(orig["bias_relu_dropout_bwd"])

    class Emu(Tapped):
        def _mm(self, a, b):
            return r16(O.blocked_matmul(a, b))

        def _wgrad(self, dy, x):
            return O.blocked_matmul(dy.reshape(-1, dy.shape[-1]).T, x.reshape(-1, x.shape[-1]))

        def _lin(self, x, w, b=None):
            t = x.dtype.type
            y = O.blocked_matmul(x.reshape(-1, x.shape[-1]), O.cast(w, t).T)
            y = y.reshape(*x.shape[:-1], -1)
            return r16(y if b is None else y + O.cast(b, t))

        def _attn_fwd(self, q, k, v, keep, t):
            s = O.blocked_matmul(q, k.swapaxes(-1, -2)) * t(1.0 / math.sqrt(q.shape[-1]))
            pr = r16(O.softmax_fwd(s, keep))
            return pr, self._join(r16(O.blocked_matmul(pr, v)))

        def _ffn_bwd(self, dy, *a):
            return r16(super()._ffn_bwd(r16(dy), *a))

        def _self_attn_bwd(self, dy1, *a):
            return r16(super()._self_attn_bwd(r16(dy1), *a))
    return Emu


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--json")
    a = ap.parse_args()
    cfg = transformer_base()
    batch = _ragged_batch(8, 64, cfg.vocab, [64, 60, 33, 64, 17, 64, 48, 64])
    train = TrainConfig(p_drop=0.1, alpha=0.1, lr=1e-3, batch_tokens=4096, seed=0,
                        cuda_graphs=False)
    eng = TrainingEngine(RunConfig(model=cfg, train=train), task=_OneBatch(batch))
    eng.setup_arena()
    step = a.steps - 1
    for s in range(step):
        eng.train_step(s)
    links = [(lk.name, lk.offset, lk.length, tuple(lk.shape)) for lk in eng.ws.links]
    p16 = H(eng.ws.params16).copy()
    M.RELU_TAP, M.GRAD_TAP = {}, {}
    eng.train_step(step)
    torch.cuda.synchronize()
    gscale = float(train.act_grad_scale)
    gtap = {k: H(v).astype(np.float64) / gscale for k, v in M.GRAD_TAP.items()}
    relu = {k: _unpack_bits(v, (8, 64, cfg.d_ff)) for k, v in M.RELU_TAP.items()}
    M.RELU_TAP = M.GRAD_TAP = None
    P = {n: O.from_half(p16[o:o + ln]).reshape(s) for n, o, ln, s in links}
    args = (batch.src, batch.tgt_in, batch.tgt_out, batch.src_len)
    kw = dict(pad_id=0, p=0.1, alpha=0.1, seed=0, step=step)
    ref = Tapped(6, 6, 512, 8, 2048, cfg.vocab, 256)
    ref.relu_inject = relu
    _, cnt, _, Gr = ref.forward_backward(P, *args, **kw)
    Emu = emulate_fp16()
    emu = Emu(6, 6, 512, 8, 2048, cfg.vocab, 256)
    emu.relu_inject = relu
    _, _, _, Ge = emu.forward_backward(P, *args, **kw)
    g16 = H(eng.ws.grads16).astype(np.float64)
    off = {n: (o, ln) for n, o, ln, _ in links}
    print("cross-query bias: column sums of the tapped dqc vs the oracle's")
    for i in range(cfg.n_dec):
        k = f"dqc:dec{i}."
        cg = gtap[k].reshape(-1, cfg.d_model).sum(0)
        cr = ref.tap[k].reshape(-1, cfg.d_model).astype(np.float64).sum(0)
        ce = emu.tap[k].reshape(-1, cfg.d_model).astype(np.float64).sum(0)
        o, ln = off[f"dec{i}.cross.bq"]
        print(f"  dec{i}: colsum(GPU dqc) {_nerr(cg, cr):.2e}  colsum(emu dqc) {_nerr(ce, cr):.2e}"
              f"  GPU cross.bq grad {_nerr(g16[o:o + ln] * cnt, cr):.2e}"
              f"  |colsum|/sum|rows| {np.linalg.norm(cr) / np.linalg.norm(np.abs(ref.tap[k].reshape(-1, cfg.d_model)).sum(0)):.2e}")
    rows = []
    for k in sorted(ref.tap, key=lambda s: (s[:2], s)):
        if k not in gtap:
            continue
        rows.append((k, _nerr(gtap[k], ref.tap[k]), _nerr(emu.tap[k], ref.tap[k])))
    print(f"step {step}: gradient taps, normwise error vs the f32 oracle")
    print(f"{'tap':16s} {'GPU':>10s} {'fp16-emu':>10s}")
    for k, eg, ee in rows:
        print(f"{k:16s} {eg:10.2e} {ee:10.2e}")
    grads = []
    for n, o, ln, s in links:
        gr = np.asarray(Gr[n], np.float64).reshape(-1) / cnt
        grads.append((n, _nerr(g16[o:o + ln], gr), _nerr(np.asarray(Ge[n]).reshape(-1) / cnt, gr)))
    grads.sort(key=lambda x: -x[1])
    print("worst parameter gradients (GPU, fp16-emu):")
    for n, eg, ee in grads[:12]:
        print(f"{n:16s} {eg:10.2e} {ee:10.2e}")
    if a.json:
        json.dump({"step": step, "taps": rows, "grads": grads}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
