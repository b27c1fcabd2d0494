"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference `ftrain` training hot path
(/root/reference/pkg/src/ftrain, abbreviated F/ below).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
leg may import this module, and only as the *checker* (or the timed CPU
baseline).  The product path (`paper_2110_05722_b200`) never imports it and
fails loudly when its CUDA library is missing.

Parity status: PINNED.  Every function here is checked against golden
input/output vectors produced by the reference itself
(tests/golden/make_golden.py imports F/ from /root/reference and writes
tests/golden/*.npz; tests/test_oracle_golden.py compares).

Dtype rule (F/kernels.py:31-36): float64 in -> float64 out; float16/float32
in -> float32 out, with row reductions accumulated in float64.
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# Counter RNG: splitmix64 over (seed, index)          F/numerics.py:19-22,133-163
# ---------------------------------------------------------------------------

M64 = (1 << 64) - 1
PHI64 = 0x9E3779B97F4A7C15
SM_A = 0xBF58476D1CE4E5B9
SM_B = 0x94D049BB133111EB


def splitmix_finalize(z: int) -> int:
    """Scalar splitmix64 finalizer (F/numerics.py:133-136)."""
    z = ((z ^ (z >> 30)) * SM_A) & M64
    z = ((z ^ (z >> 27)) * SM_B) & M64
    return z ^ (z >> 31)


def fold_seed(base: int, *tags: int) -> int:
    """derive_seed (F/numerics.py:158-163): fold tags into a 64-bit seed."""
    h = base & M64
    for t in tags:
        h = splitmix_finalize((h + PHI64 + (t & M64)) & M64)
    return h


def counter_bits53(seed: int, start: int, count: int) -> np.ndarray:
    """The 53-bit integers behind rand_uniform_array (F/numerics.py:145-155)."""
    i = np.arange(start, start + count, dtype=np.uint64)
    z = np.uint64(seed & M64) + i * np.uint64(PHI64)
    z ^= z >> np.uint64(30)
    z *= np.uint64(SM_A)
    z ^= z >> np.uint64(27)
    z *= np.uint64(SM_B)
    z ^= z >> np.uint64(31)
    return z >> np.uint64(11)


def counter_uniform(seed: int, start: int, count: int) -> np.ndarray:
    """U[0,1) draws; bit-identical to F/numerics.py:rand_uniform_array."""
    return counter_bits53(seed, start, count).astype(np.float64) / float(1 << 53)


def keep_threshold(p: float) -> int:
    """Integer form of `u >= p`: keep iff bits53 >= ceil(p * 2^53)."""
    return int(math.ceil(p * float(1 << 53)))


def dropout_keep(shape, p: float, seed: int, dtype=np.float32) -> np.ndarray:
    """make_dropout_mask (F/kernels.py:155-166): element i kept iff
    rand(seed, i) >= p over the flat row-major index; p == 0 keeps all."""
    if not 0.0 <= p < 1.0:
        raise ValueError(f"dropout probability {p} outside [0, 1)")
    n = int(np.prod(shape))
    if p == 0.0:
        return np.ones(shape, dtype=dtype)
    return (counter_uniform(seed, 0, n) >= p).astype(dtype).reshape(shape)


# ---------------------------------------------------------------------------
# binary16 narrowing                                   F/numerics.py:115-126
# ---------------------------------------------------------------------------

def to_half(x) -> np.ndarray:
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float32).astype(np.float16)


def from_half(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float16).astype(np.float32)


def half_rne_bits(f: float) -> int:
    """Independent scalar binary32 -> binary16 RNE (pins numpy's astype;
    F/numerics.py:40-85 states the same contract)."""
    u = int(np.array([f], dtype=np.float32).view(np.uint32)[0])
    s = (u >> 16) & 0x8000
    e = (u >> 23) & 0xFF
    m = u & 0x7FFFFF
    if e == 0xFF:
        return s | 0x7C00 | ((m >> 13) or (1 if m else 0))
    ue = e - 127
    if ue > 15:
        return s | 0x7C00
    if ue >= -14:
        h = s | ((ue + 15) << 10) | (m >> 13)
        r = m & 0x1FFF
        return h + (1 if (r > 0x1000 or (r == 0x1000 and (h & 1))) else 0)
    if ue < -25:
        return s
    full = m | 0x800000
    sh = 13 + (-14 - ue)
    q, r, half = full >> sh, full & ((1 << sh) - 1), 1 << (sh - 1)
    return s | (q + (1 if (r > half or (r == half and (q & 1))) else 0))


# ---------------------------------------------------------------------------
# dtype helpers                                        F/kernels.py:31-43
# ---------------------------------------------------------------------------

def ctype(*arrs):
    return np.float64 if any(a is not None and np.asarray(a).dtype == np.float64
                             for a in arrs) else np.float32


def cast(a, t):
    a = np.asarray(a)
    return a if a.dtype == t else a.astype(t)


# ---------------------------------------------------------------------------
# Forward operators
# ---------------------------------------------------------------------------

def layernorm_fwd(x, w, b, eps=1e-5):
    """Single-pass LN (F/kernels.py:235-270): mean and mean-of-squares in
    float64, sigma = sqrt(max(E[x^2]-E[x]^2, 0) + eps); returns (y, mu, sigma)."""
    x = np.asarray(x)
    t = ctype(x, w, b)
    m = x.shape[-1]
    X = x.reshape(-1, m).astype(np.float64)
    s1 = X.sum(axis=1) / m
    s2 = (X * X).sum(axis=1) / m
    var = np.maximum(s2 - s1 * s1, 0.0)
    if eps == 0.0 and np.any(var <= 0.0):
        raise ZeroDivisionError("DegenerateRow")
    sig = np.sqrt(var + eps)
    y = ((X - s1[:, None]) / sig[:, None]) * cast(w, t) + cast(b, t)
    return y.astype(t).reshape(x.shape), s1.astype(t), sig.astype(t)


def pad_keep(valid_lens, lq, lk):
    """AttentionMask('padding') (F/kernels.py:130-135): [B,1,1,Lk]."""
    lens = np.asarray(valid_lens)
    return (np.arange(lk)[None, :] < lens[:, None])[:, None, None, :]


def causal_keep(lq, lk):
    """AttentionMask('causal') (F/kernels.py:128-129)."""
    return np.arange(lk)[None, :] <= np.arange(lq)[:, None]


def softmax_fwd(x, keep=None):
    """3-step masked softmax (F/kernels.py:277-307); masked -> exact 0."""
    x = np.asarray(x)
    t = ctype(x)
    X = x.astype(np.float64)
    if keep is not None:
        X = np.where(np.broadcast_to(keep, x.shape), X, -np.inf)
    mx = X.max(axis=-1, keepdims=True)
    e = np.exp(X - mx)
    return (e / e.sum(axis=-1, keepdims=True)).astype(t)


def log_softmax_fwd(h):
    """logq = (h - max) - log sum exp (F/kernels.py:310-331)."""
    h = np.asarray(h)
    t = ctype(h)
    H = h.astype(np.float64)
    sh = H - H.max(axis=-1, keepdims=True)
    return (sh - np.log(np.exp(sh).sum(axis=-1, keepdims=True))).astype(t)


def ls_ce_fwd(logq, targets, alpha, pad_id=None):
    """(loss_sum, count) per F/kernels.py:338-360 (plugged-in smoothed CE)."""
    lq = np.asarray(logq)
    v = lq.shape[-1]
    lq = lq.reshape(-1, v)
    tg = np.asarray(targets).reshape(-1)
    ok = np.ones(tg.size, bool) if pad_id is None else tg != pad_id
    if not ok.any():
        return 0.0, 0
    rows = lq[ok].astype(np.float64)
    truth = rows[np.arange(rows.shape[0]), tg[ok]].sum()
    return float(-(1.0 - alpha) * truth - (alpha / v) * rows.sum()), int(ok.sum())


def bias_dropout_residual_fwd(x, bias, res, keep, p):
    """y = keep*(x+b)*f(1/(1-p)) + res, op order of F/kernels.py:367-382."""
    t = ctype(x, bias, res)
    y = cast(x, t) + cast(bias, t)
    if p > 0.0:
        y = (y * cast(keep, t)) * t(1.0 / (1.0 - p))
    return y + cast(res, t)


def bias_relu_dropout_fwd(x, bias, keep, p):
    """(y, relu_mask) per F/kernels.py:385-403."""
    t = ctype(x, bias)
    a = cast(x, t) + cast(bias, t)
    relu = (a > 0).astype(t)
    y = a * relu
    if p > 0.0:
        y = (y * cast(keep, t)) * t(1.0 / (1.0 - p))
    return y, relu


def embedding_fwd(emb, pos, tokens, scale, keep, p):
    """y = keep*(s*E[tok] + P[:L])/(1-p)  (F/kernels.py:203-228)."""
    t = ctype(emb, pos)
    tokens = np.asarray(tokens)
    y = cast(emb, t)[tokens] * t(scale)
    y = y + cast(pos, t)[: tokens.shape[1]][None]
    if p > 0.0:
        y = (y * cast(keep, t)) * t(1.0 / (1.0 - p))
    return y


def blocked_matmul(a, b, block=512):
    """F/kernels.py:413-447: K reduced in 512-wide blocks, fixed order."""
    k = a.shape[-1]
    acc = a[..., :block] @ b[..., :block, :]
    for k0 in range(block, k, block):
        acc = acc + a[..., k0:k0 + block] @ b[..., k0:k0 + block, :]
    return acc


# ---------------------------------------------------------------------------
# Backward operators
# ---------------------------------------------------------------------------

def layernorm_bwd(dy, x, w, mu, sigma):
    """Rearranged LN backward (F/gradients.py:103-144): two row reductions
    against alpha/beta coefficients; dw, db full-array float64 column sums."""
    dy = np.asarray(dy)
    x = np.asarray(x)
    t = ctype(dy, x, w)
    m = x.shape[-1]
    D = dy.reshape(-1, m).astype(np.float64)
    X = x.reshape(-1, m).astype(np.float64)
    mu = np.asarray(mu, np.float64).reshape(-1, 1)
    sg = np.asarray(sigma, np.float64).reshape(-1, 1)
    g = np.asarray(w, np.float64) * D
    r1 = g.sum(axis=1, keepdims=True)
    r2 = (g * X).sum(axis=1, keepdims=True)
    c = m * sg ** 3
    dx = g / sg + ((X - mu) * mu - sg * sg) / c * r1 + (mu - X) / c * r2
    xhat = (X - mu) / sg
    return (dx.astype(t).reshape(x.shape), (D * xhat).sum(axis=0).astype(t),
            D.sum(axis=0).astype(t))


def softmax_bwd(dy, q):
    """dx = q*(dy - <dy,q>)  (F/gradients.py:77-100)."""
    t = ctype(dy, q)
    D = np.asarray(dy).astype(np.float64)
    Q = np.asarray(q).astype(np.float64)
    return (Q * (D - (D * Q).sum(axis=-1, keepdims=True))).astype(t)


def ls_ce_bwd(probs, targets, alpha, pad_id=None, grad_scale=1.0):
    """dh = q - a/V - (1-a)[i==k]; pad rows 0; x grad_scale (F/gradients.py:47-74)."""
    pr = np.asarray(probs)
    v = pr.shape[-1]
    t = ctype(pr)
    P = pr.reshape(-1, v).astype(t)
    tg = np.asarray(targets).reshape(-1)
    ok = np.ones(tg.size, bool) if pad_id is None else tg != pad_id
    dh = P - t(alpha / v)
    rows = np.nonzero(ok)[0]
    dh[rows, tg[ok]] -= t(1.0 - alpha)
    dh[~ok] = 0
    if grad_scale != 1.0:
        dh[ok] *= t(grad_scale)
    return dh.reshape(pr.shape)


def bias_dropout_residual_bwd(dy, keep, p):
    """(dx, dbias, dres=dy)  F/gradients.py:147-159."""
    t = ctype(dy)
    dx = cast(dy, t).copy() if p == 0.0 else (cast(dy, t) * cast(keep, t)) * t(1.0 / (1.0 - p))
    db = dx.reshape(-1, dx.shape[-1]).astype(np.float64).sum(axis=0).astype(t)
    return dx, db, dy


def bias_relu_dropout_bwd(dy, keep, relu, p):
    """(dx, dbias)  F/gradients.py:162-172."""
    t = ctype(dy)
    dx = cast(dy, t) * cast(relu, t)
    if p > 0.0:
        dx = (dx * cast(keep, t)) * t(1.0 / (1.0 - p))
    db = dx.reshape(-1, dx.shape[-1]).astype(np.float64).sum(axis=0).astype(t)
    return dx, db


def embedding_bwd(dy, tokens, keep, p, vocab, max_len, scale, learned=True):
    """Scatter-add into the token table, per-position sum for P
    (F/gradients.py:20-44)."""
    dy = np.asarray(dy)
    t = ctype(dy)
    bsz, l, d = dy.shape
    sdy = cast(dy, t).copy() if p == 0.0 else (cast(keep, t) * dy) * t(1.0 / (1.0 - p))
    de = np.zeros((vocab, d), t)
    np.add.at(de, np.asarray(tokens).reshape(-1), sdy.reshape(-1, d))
    de *= t(scale)
    if not learned:
        return de, None
    dp = np.zeros((max_len, d), t)
    dp[:l] = sdy.sum(axis=0)
    return de, dp


# ---------------------------------------------------------------------------
# Workspace trainer                                    F/trainer.py:139-177
# ---------------------------------------------------------------------------

def adam_flat(p16, g16, m32, v32, *, lr, beta1, beta2, eps, wd, loss_scale, t):
    """Batched Adam over flat fp16 params/grads and fp32 moments, in place.
    Returns nonfinite count; on nonzero nothing is modified."""
    f = np.float32
    g = from_half(g16)
    if loss_scale != 1.0:
        g = g / f(loss_scale)
    bad = int(g.size - np.count_nonzero(np.isfinite(g)))
    if bad:
        return bad
    p = from_half(p16)
    m32[:] = f(beta1) * m32 + f(1.0 - beta1) * g
    v32[:] = f(beta2) * v32 + f(1.0 - beta2) * (g * g)
    mh = m32 / f(1.0 - beta1 ** t)
    vh = v32 / f(1.0 - beta2 ** t)
    p = p - f(lr) * (mh / (np.sqrt(vh) + f(eps)) + f(wd) * p)
    p16[:] = to_half(p)
    return 0


def sgd_flat(p16, g16, vel32, *, lr, momentum, wd, loss_scale):
    f = np.float32
    g = from_half(g16)
    if loss_scale != 1.0:
        g = g / f(loss_scale)
    bad = int(g.size - np.count_nonzero(np.isfinite(g)))
    if bad:
        return bad
    p = from_half(p16)
    if wd:
        g = g + f(wd) * p
    vel32[:] = f(momentum) * vel32 + g
    p = p - f(lr) * vel32
    p16[:] = to_half(p)
    return 0


# ---------------------------------------------------------------------------
# Static planner                                       F/memplan.py:74-101
# ---------------------------------------------------------------------------

def first_fit(lifetimes):
    """lifetimes: list of (id, size, first, last). Returns (blocks, assign)."""
    order = sorted(lifetimes, key=lambda r: (r[2], -r[1], r[0]))
    sizes, ends, assign = [], [], {}
    for tid, size, first, last in order:
        for k in range(len(sizes)):
            if ends[k] < first:
                sizes[k] = max(sizes[k], size)
                ends[k] = max(ends[k], last)
                assign[tid] = k
                break
        else:
            sizes.append(size)
            ends.append(last)
            assign[tid] = len(sizes) - 1
    return sizes, assign


# ---------------------------------------------------------------------------
# Model (fused-path semantics of F/model.py incl. dropout sites)
# ---------------------------------------------------------------------------

def model_param_shapes(n_enc, n_dec, d, dff, vocab, max_len, learned=True, tied=True):
    """Workspace layout order (F/model.py:62-97)."""
    out = [("tok_emb", (vocab, d))]
    if learned:
        out.append(("pos_emb", (max_len, d)))

    def layer(pre, dec):
        s = [(pre + "ln1.w", (d,)), (pre + "ln1.b", (d,)),
             (pre + "attn.wqkv", (3 * d, d)), (pre + "attn.bqkv", (3 * d,)),
             (pre + "attn.wo", (d, d)), (pre + "attn.bo", (d,)),
             (pre + "ln2.w", (d,)), (pre + "ln2.b", (d,))]
        if dec:
            s += [(pre + "cross.wq", (d, d)), (pre + "cross.bq", (d,)),
                  (pre + "cross.wo", (d, d)), (pre + "cross.bo", (d,)),
                  (pre + "ln3.w", (d,)), (pre + "ln3.b", (d,))]
        return s + [(pre + "ffn.w1", (dff, d)), (pre + "ffn.b1", (dff,)),
                    (pre + "ffn.w2", (d, dff)), (pre + "ffn.b2", (d,))]

    for i in range(n_enc):
        out += layer(f"enc{i}.", False)
    out += [("enc_ln.w", (d,)), ("enc_ln.b", (d,)),
            ("cross_kv.w", (2 * n_dec * d, d)), ("cross_kv.b", (2 * n_dec * d,))]
    for i in range(n_dec):
        out += layer(f"dec{i}.", True)
    out += [("dec_ln.w", (d,)), ("dec_ln.b", (d,))]
    if not tied:
        out.append(("out_proj.w", (vocab, d)))
    return out


def model_init(shapes, seed):
    """Counter-RNG init (F/model.py:100-118)."""
    params = {}
    for idx, (name, shp) in enumerate(shapes):
        leaf = name.rsplit(".", 1)[-1]
        if leaf == "w" and "ln" in name:
            params[name] = np.ones(shp, np.float32)
        elif leaf in ("b", "bqkv", "bo", "bq", "b1", "b2"):
            params[name] = np.zeros(shp, np.float32)
        else:
            u = counter_uniform(fold_seed(seed, idx), 0, int(np.prod(shp)))
            if "emb" in name or name == "out_proj.w":
                lim = 0.02 * math.sqrt(3.0)
            else:
                fo, fi = (shp[0], shp[1]) if len(shp) == 2 else (shp[0], shp[0])
                lim = math.sqrt(6.0 / (fi + fo))
            params[name] = ((2.0 * u - 1.0) * lim).astype(np.float32).reshape(shp)
    return params


def sinusoid(max_len, d, dtype=np.float32):
    """F/model.py:121-127."""
    pos = np.arange(max_len, dtype=np.float64)[:, None]
    j = np.arange(d, dtype=np.float64)[None, :]
    ang = pos / np.power(10000.0, 2.0 * np.floor(j / 2.0) / d)
    return np.where(j % 2 == 0, np.sin(ang), np.cos(ang)).astype(dtype)


class OracleTransformer:
    """Fused-graph transformer semantics (F/model.py:335-996), numpy.

    Weights: dict name -> array (any float dtype); compute dtype follows
    the F/kernels dtype rule on tok_emb.  forward_backward returns
    (loss_sum, count, correct, grads dict) with grads accumulated in the
    compute dtype exactly where F/model.py calls sink.add.
    """

    def __init__(self, n_enc, n_dec, d, heads, dff, vocab, max_len, eps=1e-5,
                 learned=True, tied=True, scale=None):
        self.n_enc, self.n_dec, self.d, self.h, self.dff = n_enc, n_dec, d, heads, dff
        self.vocab, self.max_len, self.eps = vocab, max_len, eps
        self.learned, self.tied = learned, tied
        self.scale = math.sqrt(d) if scale is None else scale
        self.relu_inject = None          # test hook, see _relu_site
        self.relu_flips = {}

    # -- attention core -------------------------------------------------------
    def _split(self, x):
        b, l, d = x.shape
        return x.reshape(b, l, self.h, d // self.h).transpose(0, 2, 1, 3)

    def _join(self, x):
        b, n, l, e = x.shape
        return x.transpose(0, 2, 1, 3).reshape(b, l, n * e)

    def _mm(self, a, b):
        return blocked_matmul(a, b)

    def _attn_fwd(self, q, k, v, keep, t):
        hd = q.shape[-1]
        s = self._mm(q, k.swapaxes(-1, -2)) * t(1.0 / math.sqrt(hd))
        pr = softmax_fwd(s, keep)
        return pr, self._join(self._mm(pr, v).astype(t))

    def _attn_bwd(self, dctxm, pr, q, k, v, t):
        hd = q.shape[-1]
        dctx = self._split(dctxm)
        ds = softmax_bwd(self._mm(dctx, v.swapaxes(-1, -2)).astype(t), pr)
        ds = ds * t(1.0 / math.sqrt(hd))
        dq = self._mm(ds, k)
        dk = self._mm(ds.swapaxes(-1, -2), q)
        dv = self._mm(pr.swapaxes(-1, -2), dctx)
        return self._join(dq).astype(t), self._join(dk).astype(t), self._join(dv).astype(t)

    def _lin(self, x, w, b=None):
        t = x.dtype.type
        y = self._mm(x.reshape(-1, x.shape[-1]), cast(w, t).T).reshape(*x.shape[:-1], -1)
        return y if b is None else y + cast(b, t)

    def _wgrad(self, dy, x):
        return self._mm(dy.reshape(-1, dy.shape[-1]).T, x.reshape(-1, x.shape[-1]))

    def _colsum(self, dy, t):
        return dy.reshape(-1, dy.shape[-1]).astype(np.float64).sum(axis=0).astype(t)

    # -- layers ---------------------------------------------------------------
    def _relu_site(self, pre, x, bias, keep, p):
        """bias_relu_dropout_fwd, optionally with injected ReLU decisions.

        relu_inject[pre] (bool [B, L, F]) replaces the oracle's own (a > 0) test,
        keeping F/kernels.py:385-403's op order for everything else; relu_flips[pre]
        records where the injected decisions differ from the oracle's own and how
        far from 0 those pre-activations were (relative to the site's RMS)."""
        inj = self.relu_inject.get(pre) if self.relu_inject else None
        if inj is None:
            return bias_relu_dropout_fwd(x, bias, keep, p)
        t = ctype(x, bias)
        a = cast(x, t) + cast(bias, t)
        own = a > 0
        diff = own != inj
        rms = float(np.sqrt(np.mean(np.square(a, dtype=np.float64))))
        self.relu_flips[pre] = (int(diff.sum()), int(diff.size),
                                float(np.abs(a[diff]).max() / rms) if diff.any() else 0.0)
        relu = inj.astype(t)
        y = a * relu
        if p > 0.0:
            y = (y * cast(keep, t)) * t(1.0 / (1.0 - p))
        return y, relu

    def _tail_fwd(self, x, wn, bn, res, p, seed, t):
        keep = dropout_keep(x.shape, p, seed, t)
        return bias_dropout_residual_fwd(x, bn, res, keep, p).astype(t), keep

    def enc_fwd(self, x, P, pre, keep_mask, p, seed, site, t):
        c = {"x": x}
        u1, c["mu1"], c["sg1"] = layernorm_fwd(x, P[pre + "ln1.w"], P[pre + "ln1.b"], self.eps)
        qkv = self._lin(u1, P[pre + "attn.wqkv"], P[pre + "attn.bqkv"])
        d = self.d
        q, k, v = (self._split(qkv[..., i * d:(i + 1) * d]) for i in range(3))
        c["probs"], ctxm = self._attn_fwd(q, k, v, keep_mask, t)
        y1, c["keep1"] = self._tail_fwd(self._lin(ctxm, P[pre + "attn.wo"]), None,
                                        P[pre + "attn.bo"], x, p, fold_seed(seed, site, 0), t)
        u2, c["mu2"], c["sg2"] = layernorm_fwd(y1, P[pre + "ln2.w"], P[pre + "ln2.b"], self.eps)
        keep2 = dropout_keep(u2.shape[:-1] + (self.dff,), p, fold_seed(seed, site, 1), t)
        z, relu = self._relu_site(pre, self._lin(u2, P[pre + "ffn.w1"]), P[pre + "ffn.b1"], keep2, p)
        y2, c["keep3"] = self._tail_fwd(self._lin(z.astype(t), P[pre + "ffn.w2"]), None,
                                        P[pre + "ffn.b2"], y1, p, fold_seed(seed, site, 2), t)
        c.update(u1=u1, qkv=qkv, ctxm=ctxm, y1=y1, u2=u2, keep2=keep2, relu=relu, z=z)
        return y2, c

    def _ffn_bwd(self, dy, c, P, pre, p, G, t, u_key, y_in_key, mu_key, sg_key, ln_name, keep_tail):
        df, db2, _ = bias_dropout_residual_bwd(dy, c[keep_tail], p)
        self._acc(G, pre + "ffn.b2", db2)
        self._acc(G, pre + "ffn.w2", self._wgrad(df, c["z"]))
        dz = self._mm(df.reshape(-1, self.d), cast(P[pre + "ffn.w2"], t)).reshape(*df.shape[:-1], -1)
        da, db1 = bias_relu_dropout_bwd(dz, c["keep2"], c["relu"], p)
        self._acc(G, pre + "ffn.b1", db1)
        self._acc(G, pre + "ffn.w1", self._wgrad(da, c[u_key]))
        du = self._mm(da.reshape(-1, self.dff), cast(P[pre + "ffn.w1"], t)).reshape(dy.shape)
        dx, dw, db = layernorm_bwd(du, c[y_in_key], P[pre + ln_name + ".w"], c[mu_key], c[sg_key])
        self._acc(G, pre + ln_name + ".w", dw)
        self._acc(G, pre + ln_name + ".b", db)
        return (dx + dy).astype(t)

    def _self_attn_bwd(self, dy1, c, P, pre, p, G, t):
        d = self.d
        dproj, dbo, _ = bias_dropout_residual_bwd(dy1, c["keep1"], p)
        self._acc(G, pre + "attn.bo", dbo)
        self._acc(G, pre + "attn.wo", self._wgrad(dproj, c["ctxm"]))
        dctxm = self._mm(dproj.reshape(-1, d), cast(P[pre + "attn.wo"], t)).reshape(dy1.shape).astype(t)
        qkv = c["qkv"]
        q, k, v = (self._split(qkv[..., i * d:(i + 1) * d]) for i in range(3))
        dq, dk, dv = self._attn_bwd(dctxm, c["probs"], q, k, v, t)
        dqkv = np.concatenate([dq, dk, dv], axis=-1)
        self._acc(G, pre + "attn.wqkv", self._wgrad(dqkv, c["u1"]))
        self._acc(G, pre + "attn.bqkv", self._colsum(dqkv, t))
        du1 = self._mm(dqkv.reshape(-1, 3 * d), cast(P[pre + "attn.wqkv"], t)).reshape(dy1.shape)
        dx, dw, db = layernorm_bwd(du1, c["x"], P[pre + "ln1.w"], c["mu1"], c["sg1"])
        self._acc(G, pre + "ln1.w", dw)
        self._acc(G, pre + "ln1.b", db)
        return (dx + dy1).astype(t)

    def enc_bwd(self, dy, c, P, pre, p, G, t):
        dy1 = self._ffn_bwd(dy, c, P, pre, p, G, t, "u2", "y1", "mu2", "sg2", "ln2", "keep3")
        return self._self_attn_bwd(dy1, c, P, pre, p, G, t)

    def dec_fwd(self, x, P, pre, kv, self_keep, cross_keep, p, seed, site, t):
        c = {"x": x}
        d = self.d
        u1, c["mu1"], c["sg1"] = layernorm_fwd(x, P[pre + "ln1.w"], P[pre + "ln1.b"], self.eps)
        qkv = self._lin(u1, P[pre + "attn.wqkv"], P[pre + "attn.bqkv"])
        q, k, v = (self._split(qkv[..., i * d:(i + 1) * d]) for i in range(3))
        c["probs"], ctxm = self._attn_fwd(q, k, v, self_keep, t)
        y1, c["keep1"] = self._tail_fwd(self._lin(ctxm, P[pre + "attn.wo"]), None,
                                        P[pre + "attn.bo"], x, p, fold_seed(seed, site, 0), t)
        u2, c["mu2"], c["sg2"] = layernorm_fwd(y1, P[pre + "ln2.w"], P[pre + "ln2.b"], self.eps)
        qc = self._lin(u2, P[pre + "cross.wq"], P[pre + "cross.bq"])
        kx, vx = kv
        c["probs_x"], ctxm_x = self._attn_fwd(self._split(qc), self._split(kx), self._split(vx),
                                              cross_keep, t)
        y2, c["keepx"] = self._tail_fwd(self._lin(ctxm_x, P[pre + "cross.wo"]), None,
                                        P[pre + "cross.bo"], y1, p, fold_seed(seed, site, 1), t)
        u3, c["mu3"], c["sg3"] = layernorm_fwd(y2, P[pre + "ln3.w"], P[pre + "ln3.b"], self.eps)
        keep2 = dropout_keep(u3.shape[:-1] + (self.dff,), p, fold_seed(seed, site, 2), t)
        z, relu = self._relu_site(pre, self._lin(u3, P[pre + "ffn.w1"]), P[pre + "ffn.b1"], keep2, p)
        y3, c["keep3"] = self._tail_fwd(self._lin(z.astype(t), P[pre + "ffn.w2"]), None,
                                        P[pre + "ffn.b2"], y2, p, fold_seed(seed, site, 3), t)
        c.update(u1=u1, qkv=qkv, ctxm=ctxm, y1=y1, u2=u2, qc=qc, ctxm_x=ctxm_x, y2=y2,
                 u3=u3, keep2=keep2, relu=relu, z=z, kv=kv)
        return y3, c

    def dec_bwd(self, dy, c, P, pre, p, G, t):
        d = self.d
        dy2 = self._ffn_bwd(dy, c, P, pre, p, G, t, "u3", "y2", "mu3", "sg3", "ln3", "keep3")
        dpx, dbx, _ = bias_dropout_residual_bwd(dy2, c["keepx"], p)
        self._acc(G, pre + "cross.bo", dbx)
        self._acc(G, pre + "cross.wo", self._wgrad(dpx, c["ctxm_x"]))
        dctx_x = self._mm(dpx.reshape(-1, d), cast(P[pre + "cross.wo"], t)).reshape(dy.shape).astype(t)
        kx, vx = c["kv"]
        dqc, dk, dv = self._attn_bwd(dctx_x, c["probs_x"], self._split(c["qc"]),
                                     self._split(kx), self._split(vx), t)
        self._acc(G, pre + "cross.wq", self._wgrad(dqc, c["u2"]))
        self._acc(G, pre + "cross.bq", self._colsum(dqc, t))
        du2 = self._mm(dqc.reshape(-1, d), cast(P[pre + "cross.wq"], t)).reshape(dy.shape)
        dx, dw, db = layernorm_bwd(du2, c["y1"], P[pre + "ln2.w"], c["mu2"], c["sg2"])
        self._acc(G, pre + "ln2.w", dw)
        self._acc(G, pre + "ln2.b", db)
        dy1 = (dx + dy2).astype(t)
        return self._self_attn_bwd(dy1, c, P, pre, p, G, t), dk, dv

    @staticmethod
    def _acc(G, name, val):
        if name in G:
            G[name] = G[name] + val
        else:
            G[name] = np.array(val, copy=True)

    # -- whole model ----------------------------------------------------------
    def forward_backward(self, P, src, tgt_in, tgt_out, src_len, *, pad_id=0, p=0.0,
                         alpha=0.0, seed=0, step=0, grad_scale=1.0, compute_grads=True,
                         capture=None):
        """F/model.py:831-996."""
        t = ctype(P["tok_emb"])
        src, tgt_in = np.asarray(src), np.asarray(tgt_in)
        tgt = np.asarray(tgt_out).reshape(-1)
        b, ls = src.shape
        lt = tgt_in.shape[1]
        pos = P["pos_emb"] if self.learned else sinusoid(self.max_len, self.d, t)
        enc_keep = pad_keep(src_len, ls, ls)
        dec_keep = causal_keep(lt, lt)
        cross_keep = pad_keep(src_len, lt, ls)

        ks = dropout_keep((b, ls, self.d), p, fold_seed(seed, step, 0), t)
        h = embedding_fwd(P["tok_emb"], pos, src, self.scale, ks, p).astype(t)
        eseed = fold_seed(seed, step, 1)
        ecache = []
        for i in range(self.n_enc):
            h, c = self.enc_fwd(h, P, f"enc{i}.", enc_keep, p, eseed, i, t)
            ecache.append(c)
        enc_in = h
        enc_out, mu_e, sg_e = layernorm_fwd(h, P["enc_ln.w"], P["enc_ln.b"], self.eps)
        kvb = self._lin(enc_out, P["cross_kv.w"], P["cross_kv.b"])
        n, d = self.n_dec, self.d
        kvs = [(kvb[..., i * d:(i + 1) * d], kvb[..., (n + i) * d:(n + i + 1) * d]) for i in range(n)]

        kt = dropout_keep((b, lt, d), p, fold_seed(seed, step, 2), t)
        g = embedding_fwd(P["tok_emb"], pos, tgt_in, self.scale, kt, p).astype(t)
        dseed = fold_seed(seed, step, 3)
        dcache = []
        for i in range(self.n_dec):
            g, c = self.dec_fwd(g, P, f"dec{i}.", kvs[i], dec_keep, cross_keep, p, dseed, i, t)
            dcache.append(c)
        dec_in = g
        dec_out, mu_d, sg_d = layernorm_fwd(g, P["dec_ln.w"], P["dec_ln.b"], self.eps)
        W = P["tok_emb"] if self.tied else P["out_proj.w"]
        logits = self._mm(dec_out.reshape(-1, d), cast(W, t).T).astype(t)
        logq = log_softmax_fwd(logits)
        loss, count = ls_ce_fwd(logq, tgt, alpha, pad_id)
        ok = tgt != pad_id
        correct = int((np.argmax(logq, axis=-1)[ok] == tgt[ok]).sum())
        if capture is not None:
            capture["logq"] = logq.reshape(b, lt, -1).copy()
        if not compute_grads:
            return loss, count, correct, None

        G = {}
        dl = ls_ce_bwd(np.exp(logq), tgt, alpha, pad_id, grad_scale).astype(t)
        wname = "tok_emb" if self.tied else "out_proj.w"
        ddec = self._mm(dl, cast(W, t)).reshape(b, lt, d).astype(t)
        self._acc(G, wname, self._mm(dl.T, dec_out.reshape(-1, d)))
        dg, dw, db = layernorm_bwd(ddec, dec_in, P["dec_ln.w"], mu_d, sg_d)
        self._acc(G, "dec_ln.w", dw)
        self._acc(G, "dec_ln.b", db)
        dks, dvs = [None] * n, [None] * n
        for i in reversed(range(n)):
            dg, dks[i], dvs[i] = self.dec_bwd(dg, dcache[i], P, f"dec{i}.", p, G, t)
        de, dp = embedding_bwd(dg, tgt_in, kt, p, self.vocab, self.max_len, self.scale, self.learned)
        self._acc(G, "tok_emb", de)
        if dp is not None:
            self._acc(G, "pos_emb", dp)
        dkv = np.concatenate(dks + dvs, axis=-1).astype(t)
        denc = self._mm(dkv.reshape(-1, 2 * n * d), cast(P["cross_kv.w"], t)).reshape(enc_out.shape).astype(t)
        self._acc(G, "cross_kv.w", self._wgrad(dkv, enc_out))
        self._acc(G, "cross_kv.b", self._colsum(dkv, t))
        dh, dw, db = layernorm_bwd(denc, enc_in, P["enc_ln.w"], mu_e, sg_e)
        self._acc(G, "enc_ln.w", dw)
        self._acc(G, "enc_ln.b", db)
        for i in reversed(range(self.n_enc)):
            dh = self.enc_bwd(dh, ecache[i], P, f"enc{i}.", p, G, t)
        de, dp = embedding_bwd(dh, src, ks, p, self.vocab, self.max_len, self.scale, self.learned)
        self._acc(G, "tok_emb", de)
        if dp is not None:
            self._acc(G, "pos_emb", dp)
        return loss, count, correct, G


def train_step_flat(model: OracleTransformer, shapes, p16, m32, v32, batch, *, p_drop, alpha,
                    seed, step, lr, beta1=0.9, beta2=0.999, eps_opt=1e-8, wd=0.0,
                    loss_scale=1.0, t):
    """One engine step (F/engine.py:130-169): fp16 workspace views ->
    forward/backward -> grad_acc * f32(loss_scale/count) -> narrow -> Adam.
    Returns (loss_sum, count, correct, applied)."""
    P, off = {}, 0
    for name, shp in shapes:
        n = int(np.prod(shp))
        P[name] = p16[off:off + n].reshape(shp)
        off += n
    src, tgt_in, tgt_out, src_len, pad_id = batch
    loss, count, correct, G = model.forward_backward(
        P, src, tgt_in, tgt_out, src_len, pad_id=pad_id, p=p_drop, alpha=alpha, seed=seed,
        step=step)
    if not np.isfinite(loss):
        return loss, count, correct, False
    acc = np.concatenate([np.asarray(G[name], np.float32).reshape(-1) for name, _ in shapes])
    acc *= np.float32(loss_scale / max(count, 1))
    g16 = to_half(acc)
    bad = adam_flat(p16, g16, m32, v32, lr=lr, beta1=beta1, beta2=beta2, eps=eps_opt, wd=wd,
                    loss_scale=loss_scale, t=t)
    return loss, count, correct, bad == 0


# ---------------------------------------------------------------------------
# BERT-shaped encoder + tied MLM criterion (BASELINE.json configs[3]).  Not a
# reference model: composed only from the pinned pieces above (embedding,
# encoder layer, LayerNorm, log-softmax, label-smoothed CE) in the order
# F/model.py:831-996 applies them to the encoder half; non-MLM positions carry
# the pad target.  Its parity rests on those pieces' golden pins.
# ---------------------------------------------------------------------------

def encoder_param_shapes(n_enc, d, dff, vocab, max_len, learned=True):
    full = model_param_shapes(n_enc, 0, d, dff, vocab, max_len, learned)
    keep = [s for s in full if not s[0].startswith(("cross_kv.", "dec_ln."))]
    return keep


class OracleEncoderMLM(OracleTransformer):
    def __init__(self, n_enc, d, heads, dff, vocab, max_len, eps=1e-5, **kw):
        super().__init__(n_enc, 0, d, heads, dff, vocab, max_len, eps, **kw)

    def forward_backward(self, P, src, tgt_out, src_len, *, pad_id=0, p=0.0, alpha=0.0, seed=0,
                         step=0, grad_scale=1.0, compute_grads=True):
        t = ctype(P["tok_emb"])
        src = np.asarray(src)
        tgt = np.asarray(tgt_out).reshape(-1)
        b, ls = src.shape
        d = self.d
        pos = P["pos_emb"] if self.learned else sinusoid(self.max_len, d, t)
        enc_keep = pad_keep(src_len, ls, ls)
        ks = dropout_keep((b, ls, d), p, fold_seed(seed, step, 0), t)
        h = embedding_fwd(P["tok_emb"], pos, src, self.scale, ks, p).astype(t)
        eseed = fold_seed(seed, step, 1)
        ecache = []
        for i in range(self.n_enc):
            h, c = self.enc_fwd(h, P, f"enc{i}.", enc_keep, p, eseed, i, t)
            ecache.append(c)
        enc_in = h
        enc_out, mu_e, sg_e = layernorm_fwd(h, P["enc_ln.w"], P["enc_ln.b"], self.eps)
        W = P["tok_emb"]
        logits = self._mm(enc_out.reshape(-1, d), cast(W, t).T).astype(t)
        logq = log_softmax_fwd(logits)
        loss, count = ls_ce_fwd(logq, tgt, alpha, pad_id)
        ok = tgt != pad_id
        correct = int((np.argmax(logq, axis=-1)[ok] == tgt[ok]).sum())
        if not compute_grads:
            return loss, count, correct, None
        G = {}
        dl = ls_ce_bwd(np.exp(logq), tgt, alpha, pad_id, grad_scale).astype(t)
        denc = self._mm(dl, cast(W, t)).reshape(b, ls, d).astype(t)
        self._acc(G, "tok_emb", self._mm(dl.T, enc_out.reshape(-1, d)))
        dh, dw, db = layernorm_bwd(denc, enc_in, P["enc_ln.w"], mu_e, sg_e)
        self._acc(G, "enc_ln.w", dw)
        self._acc(G, "enc_ln.b", db)
        for i in reversed(range(self.n_enc)):
            dh = self.enc_bwd(dh, ecache[i], P, f"enc{i}.", p, G, t)
        de, dpos = embedding_bwd(dh, src, ks, p, self.vocab, self.max_len, self.scale, self.learned)
        self._acc(G, "tok_emb", de)
        if dpos is not None:
            self._acc(G, "pos_emb", dpos)
        return loss, count, correct, G
