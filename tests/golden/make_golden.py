"""Generate golden input/output vectors from the REFERENCE implementation.

Run in the build container (needs /root/reference, read-only):

    python tests/golden/make_golden.py

It imports the reference package `ftrain` from /root/reference/pkg/src,
runs its own operators on seeded inputs and writes tests/golden/*.npz.
The GPU box never has /root/reference; tests only read the .npz files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _import_ref():
    sys.dont_write_bytecode = True  # the reference tree is read-only
    sys.path.insert(0, REF_SRC)
    import ftrain  # noqa: F401
    from ftrain import gradients as G
    from ftrain import kernels as K
    from ftrain import memplan, model, numerics, trainer
    return K, G, numerics, trainer, memplan, model


def main():
    K, G, N, T, MP, M = _import_ref()
    rng = np.random.default_rng(20211012)
    out = {}

    # --- RNG / masks (F/numerics.py:139-163, F/kernels.py:155-166) -------------
    seeds = [0, 1, 77, 2**63 + 12345, 2**64 - 1]
    for i, s in enumerate(seeds):
        out[f"rng_u_{i}"] = N.rand_uniform_array(s, 1000 * i, 4099)
        out[f"rng_seed_{i}"] = np.array([s], dtype=np.uint64)
        out[f"rng_start_{i}"] = np.array([1000 * i], dtype=np.int64)
    derived = []
    for s in seeds:
        for tags in [(0,), (3, 1), (7, 2, 5), (2**40, 9)]:
            derived.append([s, len(tags), *tags, *([0] * (3 - len(tags))), N.derive_seed(s, *tags)])
    out["derive_rows"] = np.array(derived, dtype=np.uint64)
    for j, (shape, p, s) in enumerate([((3, 5, 7), 0.1, 5), ((64, 33), 0.5, 77),
                                       ((2, 2, 2), 0.0, 1), ((1000,), 0.9, 2**63 + 1)]):
        m = K.make_dropout_mask(shape, p, s, np.float32)
        out[f"mask_{j}_keep"] = m.keep
        out[f"mask_{j}_p"] = np.array([p])
        out[f"mask_{j}_seed"] = np.array([s], dtype=np.uint64)

    # --- fp16 narrowing spot values ---------------------------------------------
    vals = np.array([1.0, 0.1, 65504.0, 65519.99, 65520.0, -70000.0, 2.0**-24, 2.0**-25,
                     3 * 2.0**-26, 6.1e-5, 1e-8, -0.0, np.inf, -np.inf, 0.3333333],
                    dtype=np.float32)
    out["half_in"] = vals
    out["half_bits"] = N.narrow_f32(vals).view(np.uint16)

    # --- layernorm (F/kernels.py:235-270, F/gradients.py:103-144) ---------------
    for dt, tag in [(np.float64, "f64"), (np.float32, "f32"), (np.float16, "f16")]:
        x = (rng.normal(size=(37, 48)) * 3 + 1).astype(dt)
        w = rng.normal(size=48).astype(dt)
        b = rng.normal(size=48).astype(dt)
        dy = rng.normal(size=(37, 48)).astype(dt)
        y, c = K.layernorm_forward(x, w, b, 1e-5)
        dx, dw, db = G.layernorm_backward(dy, x, w, c)
        out.update({f"ln_{tag}_x": x, f"ln_{tag}_w": w, f"ln_{tag}_b": b, f"ln_{tag}_dy": dy,
                    f"ln_{tag}_y": y, f"ln_{tag}_mu": c.mu, f"ln_{tag}_sigma": c.sigma,
                    f"ln_{tag}_dx": dx, f"ln_{tag}_dw": dw, f"ln_{tag}_db": db})
    xs = rng.normal(0, 1, (64, 16)) + 1000.0
    _, cs = K.layernorm_forward(xs, np.ones(16), np.zeros(16), eps=0.0)
    out["ln_shift_x"], out["ln_shift_sigma"] = xs, cs.sigma

    # --- softmax / log-softmax (F/kernels.py:277-331, F/gradients.py:77-100) ----
    for dt, tag in [(np.float64, "f64"), (np.float32, "f32")]:
        x = (rng.normal(size=(2, 3, 5, 7)) * 4).astype(dt)
        dy = rng.normal(size=(2, 3, 5, 7)).astype(dt)
        lens = np.array([7, 3])
        for mk, mask in [("none", None), ("pad", K.AttentionMask("padding", lens)),
                         ("causal", K.AttentionMask("causal"))]:
            y, c = K.softmax_forward(x, mask=mask)
            out[f"sm_{tag}_{mk}_y"] = y
            out[f"sm_{tag}_{mk}_dx"] = G.softmax_backward(dy, c)
        out[f"sm_{tag}_x"], out[f"sm_{tag}_dy"], out[f"sm_{tag}_lens"] = x, dy, lens
        h = (rng.normal(size=(9, 31)) * 5).astype(dt)
        out[f"lsm_{tag}_h"], out[f"lsm_{tag}_y"] = h, K.log_softmax_forward(h)

    # --- criterion (F/kernels.py:338-360, F/gradients.py:47-74) -----------------
    for dt, tag in [(np.float64, "f64"), (np.float32, "f32")]:
        h = (rng.normal(size=(12, 29)) * 2).astype(dt)
        tg = rng.integers(0, 29, 12)
        tg[[1, 5]] = 0
        for a in (0.0, 0.1, 1.0):
            logq = K.log_softmax_forward(h)
            loss, cnt = K.ls_cross_entropy_forward(logq, tg, a, pad_id=0)
            pr, _ = K.softmax_forward(h)
            dh = G.ls_cross_entropy_backward(pr, tg, a, pad_id=0, grad_scale=0.25)
            out[f"ce_{tag}_{a}_loss"] = np.array([loss, cnt])
            out[f"ce_{tag}_{a}_dh"] = dh
        out[f"ce_{tag}_h"], out[f"ce_{tag}_t"] = h, tg

    # --- fused elementwise tails (F/kernels.py:367-403, F/gradients.py:147-172) --
    for dt, tag in [(np.float64, "f64"), (np.float32, "f32"), (np.float16, "f16")]:
        x = rng.normal(size=(4, 6, 40)).astype(dt)
        res = rng.normal(size=(4, 6, 40)).astype(dt)
        bias = rng.normal(size=40).astype(dt)
        dy = rng.normal(size=(4, 6, 40)).astype(dt)
        y, mk = K.bias_dropout_residual(x, bias, res, 0.3, seed=1234)
        dx, db, _ = G.bias_dropout_residual_backward(dy, mk)
        y2, mk2, rl = K.bias_relu_dropout(x, bias, 0.25, seed=99)
        dx2, db2 = G.bias_relu_dropout_backward(dy, mk2, rl)
        out.update({f"bdr_{tag}_x": x, f"bdr_{tag}_res": res, f"bdr_{tag}_bias": bias,
                    f"bdr_{tag}_dy": dy, f"bdr_{tag}_y": y, f"bdr_{tag}_keep": mk.keep,
                    f"bdr_{tag}_dx": dx, f"bdr_{tag}_db": db,
                    f"brd_{tag}_y": y2, f"brd_{tag}_keep": mk2.keep, f"brd_{tag}_relu": rl,
                    f"brd_{tag}_dx": dx2, f"brd_{tag}_db": db2})

    # --- embedding (F/kernels.py:203-228, F/gradients.py:20-44) -----------------
    for dt, tag in [(np.float64, "f64"), (np.float32, "f32")]:
        emb = rng.normal(size=(23, 16)).astype(dt)
        pos = rng.normal(size=(9, 16)).astype(dt)
        tok = rng.integers(0, 23, (3, 7))
        tok[0, :3] = 5  # repeated token
        cfg = K.EmbeddingConfig(scale=4.0, vocab=23, max_len=9)
        y, mk = K.embedding_forward(emb, pos, tok, cfg, 0.2, seed=31)
        dy = rng.normal(size=y.shape).astype(dt)
        de, dp = G.embedding_backward(dy, tok, mk, cfg)
        out.update({f"emb_{tag}_E": emb, f"emb_{tag}_P": pos, f"emb_{tag}_tok": tok,
                    f"emb_{tag}_y": y, f"emb_{tag}_keep": mk.keep, f"emb_{tag}_dy": dy,
                    f"emb_{tag}_dE": de, f"emb_{tag}_dP": dp})

    # --- workspace trainer (F/trainer.py:101-181) --------------------------------
    for algo in ("adam", "sgd"):
        p0 = (rng.normal(size=777) * 2).astype(np.float32)
        ws = T.workspace_pack([("a", p0[:500].reshape(20, 25)), ("b", p0[500:])], algo)
        cfg = T.OptimConfig(algorithm=algo, lr=3e-3, weight_decay=0.01, momentum=0.9,
                            loss_scale=8.0)
        ws.m32[:] = (rng.normal(size=777) * 0.01).astype(np.float32)
        if algo == "adam":
            ws.v32[:] = rng.uniform(0, 0.01, 777).astype(np.float32)
        out[f"tr_{algo}_p0"] = ws.params16.copy()
        out[f"tr_{algo}_m0"] = ws.m32.copy()
        if algo == "adam":
            out[f"tr_{algo}_v0"] = ws.v32.copy()
        gs = []
        for t in range(1, 6):
            g = T.narrow_f32((rng.normal(size=777) * 0.5 * t).astype(np.float32))
            if t == 4:
                g[17] = np.float16(np.inf)  # skipped step
            gs.append(g)
            ws.grads16[:] = g
            rep = T.optimizer_step(ws, cfg, t)
            out[f"tr_{algo}_p{t}"] = ws.params16.copy()
            out[f"tr_{algo}_applied{t}"] = np.array([rep.applied, rep.nonfinite])
        out[f"tr_{algo}_g"] = np.stack(gs)
        out[f"tr_{algo}_mfinal"] = ws.m32.copy()
        if algo == "adam":
            out[f"tr_{algo}_vfinal"] = ws.v32.copy()

    # --- memory planner (F/memplan.py:74-101) ------------------------------------
    lts = []
    for i in range(40):
        f = int(rng.integers(0, 60))
        lts.append((i, int(rng.integers(1, 500)), f, f + int(rng.integers(0, 20))))
    p = MP.plan([MP.Lifetime(*x) for x in lts])
    out["plan_in"] = np.array(lts)
    out["plan_blocks"] = np.array(p.blocks)
    out["plan_assign"] = np.array([p.assignment[i] for i in range(40)])

    np.savez_compressed(os.path.join(OUT, "ops.npz"), **out)

    # --- tiny model, fused path with dropout (F/model.py:831-996) ----------------
    mout = {}
    cfg = M.ModelConfig(n_enc=2, n_dec=2, d_model=16, n_heads=4, d_ff=24, vocab=19, max_len=8)
    tf = M.Transformer(cfg)
    init = tf.init_params(seed=3)
    for name in tf.param_names:
        mout[f"init_{name}"] = init[name]
    brng = np.random.default_rng(5)
    b, l = 3, 6
    src = brng.integers(2, 19, (b, l))
    tgt_in = brng.integers(2, 19, (b, l))
    tgt_out = brng.integers(2, 19, (b, l))
    src_len = np.array([6, 4, 2])
    tgt_out[2, 4:] = 0
    tgt_in[2, 5:] = 0
    mout.update(src=src, tgt_in=tgt_in, tgt_out=tgt_out, src_len=src_len)
    for dt, tag in [(np.float64, "f64"), (np.float32, "f32")]:
        P = {k: v.astype(dt) for k, v in init.items()}
        sink = M.GradSink()
        cap = {}
        o = tf.forward_backward(P, M.Batch(src, tgt_in, tgt_out, src_len, 0), p_drop=0.2,
                                alpha=0.1, seed=11, step=4, sink=sink, capture=cap)
        mout[f"{tag}_out"] = np.array([o.loss_sum, o.token_count, o.correct])
        mout[f"{tag}_logq"] = cap["logq"]
        for k, v in sink.store.items():
            mout[f"{tag}_g_{k}"] = v
    # engine-style fp16 workspace steps (F/engine.py:130-169)
    ws = T.workspace_pack([(n, init[n]) for n in tf.param_names], "adam")
    pv = ws.param_views()
    acc = np.zeros(ws.n_elements, np.float32)
    gv = {lk.name: acc[lk.offset:lk.offset + lk.length].reshape(lk.shape) for lk in ws.links}
    ocfg = T.OptimConfig(lr=2e-3, loss_scale=4.0)
    for step in range(3):
        acc.fill(0)
        o = tf.forward_backward(pv, M.Batch(src, tgt_in, tgt_out, src_len, 0), p_drop=0.1,
                                alpha=0.1, seed=7, step=step, sink=M._ViewSink(gv))
        acc *= np.float32(ocfg.loss_scale / o.token_count)
        ws.grads16[:] = N.narrow_f32(acc)
        mout[f"eng_g16_{step}"] = ws.grads16.copy()
        T.adam_step(ws, ocfg, step + 1)
        T.zero_grads(ws)
        mout[f"eng_p16_{step}"] = ws.params16.copy()
        mout[f"eng_loss_{step}"] = np.array([o.loss_sum, o.token_count, o.correct])
    np.savez_compressed(os.path.join(OUT, "model.npz"), **mout)

    # --- default-config training trajectory (F/engine.py, copy task, 400 steps) --
    from ftrain.config import RunConfig
    from ftrain.engine import TrainingEngine
    run = RunConfig()
    run.train.p_drop = 0.1
    eng = TrainingEngine(run)
    eng.setup_arena()
    losses = [eng.train_step(s).loss for s in range(400)]
    np.savez_compressed(os.path.join(OUT, "traj.npz"), losses=np.array(losses),
                        eval_acc=np.array([eng.evaluate()]))
    print("wrote", os.path.join(OUT, "ops.npz"), os.path.join(OUT, "model.npz"),
          os.path.join(OUT, "traj.npz"))


if __name__ == "__main__":
    main()
