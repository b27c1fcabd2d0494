"""Pin the CPU oracle (oracle/lsport.py) to golden vectors the reference produced.

CPU-only; reads tests/golden/*.npz written by tests/golden/make_golden.py.
"""

import numpy as np
import pytest

from conftest import rel_err
from oracle import lsport as O


def test_rng_uniform_bit_identical(golden_ops):
    g = golden_ops
    for i in range(5):
        seed = int(g[f"rng_seed_{i}"][0])
        start = int(g[f"rng_start_{i}"][0])
        u = O.counter_uniform(seed, start, 4099)
        assert np.array_equal(u.view(np.uint64), g[f"rng_u_{i}"].view(np.uint64))


def test_derive_seed_bit_identical(golden_ops):
    for row in golden_ops["derive_rows"]:
        s, n = int(row[0]), int(row[1])
        tags = [int(t) for t in row[2:2 + n]]
        assert O.fold_seed(s, *tags) == int(row[5])


def test_dropout_masks_and_integer_threshold(golden_ops):
    g = golden_ops
    for j in range(4):
        keep = g[f"mask_{j}_keep"]
        p = float(g[f"mask_{j}_p"][0])
        seed = int(g[f"mask_{j}_seed"][0])
        mine = O.dropout_keep(keep.shape, p, seed)
        assert np.array_equal(mine, keep)
        if p > 0:
            bits = O.counter_bits53(seed, 0, keep.size)
            assert np.array_equal((bits >= np.uint64(O.keep_threshold(p))).reshape(keep.shape),
                                  keep.astype(bool))


def test_half_narrowing(golden_ops):
    g = golden_ops
    assert np.array_equal(O.to_half(g["half_in"]).view(np.uint16), g["half_bits"])
    for v, b in zip(g["half_in"], g["half_bits"]):
        assert O.half_rne_bits(float(v)) == int(b)


@pytest.mark.parametrize("tag,tol", [("f64", 1e-12), ("f32", 1e-6), ("f16", 1e-6)])
def test_layernorm(golden_ops, tag, tol):
    g = golden_ops
    y, mu, sg = O.layernorm_fwd(g[f"ln_{tag}_x"], g[f"ln_{tag}_w"], g[f"ln_{tag}_b"], 1e-5)
    assert y.dtype == g[f"ln_{tag}_y"].dtype
    assert rel_err(y, g[f"ln_{tag}_y"], 1.0) < tol
    assert rel_err(sg, g[f"ln_{tag}_sigma"]) < tol
    dx, dw, db = O.layernorm_bwd(g[f"ln_{tag}_dy"], g[f"ln_{tag}_x"], g[f"ln_{tag}_w"],
                                 g[f"ln_{tag}_mu"], g[f"ln_{tag}_sigma"])
    assert rel_err(dx, g[f"ln_{tag}_dx"], 1.0) < tol
    assert rel_err(dw, g[f"ln_{tag}_dw"], 1.0) < tol
    assert rel_err(db, g[f"ln_{tag}_db"], 1.0) < tol
    _, _, s = O.layernorm_fwd(g["ln_shift_x"], np.ones(16), np.zeros(16), 0.0)
    assert rel_err(s, g["ln_shift_sigma"]) < 1e-9


@pytest.mark.parametrize("tag,tol", [("f64", 1e-12), ("f32", 1e-6)])
def test_softmax_family(golden_ops, tag, tol):
    g = golden_ops
    x, dy, lens = g[f"sm_{tag}_x"], g[f"sm_{tag}_dy"], g[f"sm_{tag}_lens"]
    masks = {"none": None, "pad": O.pad_keep(lens, 5, 7), "causal": O.causal_keep(5, 7)}
    for mk, keep in masks.items():
        y = O.softmax_fwd(x, keep)
        assert rel_err(y, g[f"sm_{tag}_{mk}_y"], 1.0) < tol
        assert rel_err(O.softmax_bwd(dy, y), g[f"sm_{tag}_{mk}_dx"], 1.0) < tol
    assert rel_err(O.log_softmax_fwd(g[f"lsm_{tag}_h"]), g[f"lsm_{tag}_y"], 1.0) < tol


@pytest.mark.parametrize("tag,tol", [("f64", 1e-12), ("f32", 1e-6)])
def test_criterion(golden_ops, tag, tol):
    g = golden_ops
    h, tg = g[f"ce_{tag}_h"], g[f"ce_{tag}_t"]
    for a in (0.0, 0.1, 1.0):
        loss, cnt = O.ls_ce_fwd(O.log_softmax_fwd(h), tg, a, pad_id=0)
        want = g[f"ce_{tag}_{a}_loss"]
        assert cnt == int(want[1])
        assert abs(loss - want[0]) <= tol * max(1.0, abs(want[0]))
        dh = O.ls_ce_bwd(O.softmax_fwd(h), tg, a, pad_id=0, grad_scale=0.25)
        assert rel_err(dh, g[f"ce_{tag}_{a}_dh"], 1.0) < tol


@pytest.mark.parametrize("tag", ["f64", "f32", "f16"])
def test_elementwise_tails(golden_ops, tag):
    g = golden_ops
    x, res, bias, dy = (g[f"bdr_{tag}_{k}"] for k in ("x", "res", "bias", "dy"))
    keep = O.dropout_keep(x.shape, 0.3, 1234, g[f"bdr_{tag}_keep"].dtype)
    assert np.array_equal(keep, g[f"bdr_{tag}_keep"])
    y = O.bias_dropout_residual_fwd(x, bias, res, keep, 0.3)
    assert np.array_equal(y, g[f"bdr_{tag}_y"])          # same op order: bit-exact
    dx, db, dres = O.bias_dropout_residual_bwd(dy, keep, 0.3)
    assert np.array_equal(dx, g[f"bdr_{tag}_dx"]) and dres is dy
    assert np.array_equal(db, g[f"bdr_{tag}_db"])
    keep2 = O.dropout_keep(x.shape, 0.25, 99, g[f"brd_{tag}_keep"].dtype)
    y2, relu = O.bias_relu_dropout_fwd(x, bias, keep2, 0.25)
    assert np.array_equal(y2, g[f"brd_{tag}_y"]) and np.array_equal(relu, g[f"brd_{tag}_relu"])
    dx2, db2 = O.bias_relu_dropout_bwd(dy, keep2, relu, 0.25)
    assert np.array_equal(dx2, g[f"brd_{tag}_dx"]) and np.array_equal(db2, g[f"brd_{tag}_db"])


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_embedding(golden_ops, tag):
    g = golden_ops
    E, P, tok, dy = (g[f"emb_{tag}_{k}"] for k in ("E", "P", "tok", "dy"))
    keep = O.dropout_keep((3, 7, 16), 0.2, 31, E.dtype if tag == "f64" else np.float32)
    assert np.array_equal(keep, g[f"emb_{tag}_keep"])
    y = O.embedding_fwd(E, P, tok, 4.0, keep, 0.2)
    assert np.array_equal(y, g[f"emb_{tag}_y"])
    de, dp = O.embedding_bwd(dy, tok, keep, 0.2, 23, 9, 4.0)
    assert np.array_equal(de, g[f"emb_{tag}_dE"]) and np.array_equal(dp, g[f"emb_{tag}_dP"])


@pytest.mark.parametrize("algo", ["adam", "sgd"])
def test_trainer_bit_exact(golden_ops, algo):
    g = golden_ops
    p16 = g[f"tr_{algo}_p0"].copy()
    m = g[f"tr_{algo}_m0"].copy()
    v = g[f"tr_{algo}_v0"].copy() if algo == "adam" else None
    for t in range(1, 6):
        g16 = g[f"tr_{algo}_g"][t - 1]
        if algo == "adam":
            bad = O.adam_flat(p16, g16, m, v, lr=3e-3, beta1=0.9, beta2=0.999, eps=1e-8,
                              wd=0.01, loss_scale=8.0, t=t)
        else:
            bad = O.sgd_flat(p16, g16, m, lr=3e-3, momentum=0.9, wd=0.01, loss_scale=8.0)
        applied, nonfinite = g[f"tr_{algo}_applied{t}"]
        assert (bad == 0) == bool(applied) and bad == nonfinite
        assert np.array_equal(p16.view(np.uint16), g[f"tr_{algo}_p{t}"].view(np.uint16))
    assert np.array_equal(m, g[f"tr_{algo}_mfinal"])
    if v is not None:
        assert np.array_equal(v, g[f"tr_{algo}_vfinal"])


def test_planner(golden_ops):
    g = golden_ops
    blocks, assign = O.first_fit([tuple(int(v) for v in r) for r in g["plan_in"]])
    assert blocks == list(g["plan_blocks"])
    assert [assign[i] for i in range(40)] == list(g["plan_assign"])


def _tiny():
    return O.OracleTransformer(2, 2, 16, 4, 24, 19, 8)


def _params(gm, dt):
    shapes = O.model_param_shapes(2, 2, 16, 24, 19, 8)
    init = O.model_init(shapes, seed=3)
    for name, _ in shapes:
        assert np.array_equal(init[name], gm[f"init_{name}"]), name
    return shapes, {k: v.astype(dt) for k, v in init.items()}


@pytest.mark.parametrize("tag,dt,tol", [("f64", np.float64, 1e-10), ("f32", np.float32, 2e-5)])
def test_model_forward_backward(golden_model, tag, dt, tol):
    gm = golden_model
    shapes, P = _params(gm, dt)
    cap = {}
    loss, cnt, cor, G = _tiny().forward_backward(
        P, gm["src"], gm["tgt_in"], gm["tgt_out"], gm["src_len"], pad_id=0, p=0.2, alpha=0.1,
        seed=11, step=4, capture=cap)
    want = gm[f"{tag}_out"]
    assert abs(loss - want[0]) <= tol * abs(want[0])
    assert cnt == want[1] and cor == want[2]
    assert rel_err(cap["logq"], gm[f"{tag}_logq"], 1.0) < tol
    for name, _ in shapes:
        ref = gm[f"{tag}_g_{name}"]
        scale = max(1.0, float(np.abs(ref).max()))
        assert np.abs(G[name] - ref).max() <= tol * scale, name


def test_engine_steps_fp16(golden_model):
    gm = golden_model
    shapes, P = _params(gm, np.float32)
    p16 = np.concatenate([O.to_half(P[n].reshape(-1)) for n, _ in shapes])
    m = np.zeros(p16.size, np.float32)
    v = np.zeros(p16.size, np.float32)
    model = _tiny()
    batch = (gm["src"], gm["tgt_in"], gm["tgt_out"], gm["src_len"], 0)
    for step in range(3):
        loss, cnt, cor, applied = O.train_step_flat(
            model, shapes, p16, m, v, batch, p_drop=0.1, alpha=0.1, seed=7, step=step,
            lr=2e-3, loss_scale=4.0, t=step + 1)
        want = gm[f"eng_loss_{step}"]
        assert abs(loss - want[0]) <= 1e-5 * abs(want[0]) and applied
        # fp16 params after the update: identical except where the fp32 grads
        # differ in the last bit before narrowing (accumulation order).
        ref = gm[f"eng_p16_{step}"].astype(np.float32)
        mine = p16.astype(np.float32)
        assert np.mean(mine != ref) < 1e-3
        assert np.abs(mine - ref).max() <= 2e-3 * max(1.0, np.abs(ref).max())
        p16[:] = gm[f"eng_p16_{step}"]   # re-sync so steps stay comparable
