"""The reference's own unit tests, restated against the CUDA path.

Each test below restates one test of /root/reference/pkg/tests (written T/):
test_kernels.py, test_gradients.py and test_trainer.py, cited per test.  The
mirror modules are called through tests/numpy_shim.py exactly as the reference
tests call `ftrain.kernels` / `ftrain.gradients` / `ftrain.trainer`: numpy in,
numpy out, in-place `out=` / `accumulate_into=` arrays.  The checked numbers,
known answers and tolerances are the reference's; only the thread-count tests
become determinism tests (the device path has no CPU thread pool: run twice,
compare bits).  The reference's own oracle helpers are replaced by the pinned
oracle (oracle/lsport.py) or by a direct formula written in the test.

Where the reference's tolerance assumes float64 arithmetic the test runs the
f64 kernels (the mirror keeps the reference's dtype rule: f64 in -> f64 out).
"""

import math

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st
from hypothesis.extra.numpy import arrays

from numpy_shim import NumpyAPI, host
from oracle import lsport as O

pytestmark = pytest.mark.gpu

kernels = pytest.importorskip("paper_2110_05722_b200.kernels")
from paper_2110_05722_b200 import gradients as _gradients  # noqa: E402
from paper_2110_05722_b200 import numerics as _numerics  # noqa: E402
from paper_2110_05722_b200 import trainer as T  # noqa: E402
from paper_2110_05722_b200.errors import (AllMaskedRow, ConfigError, DegenerateRow,  # noqa: E402
                                          DuplicateName, SequenceTooLong, ShapeMismatch,
                                          TokenOutOfRange)
from paper_2110_05722_b200.kernels import (AttentionMask, DropoutMask,  # noqa: E402
                                           EmbeddingConfig, SoftmaxCache)

K = NumpyAPI(kernels)
G = NumpyAPI(_gradients)

FEW = settings(max_examples=25, deadline=None)


@pytest.fixture(autouse=True)
def _fresh_autotune_cache():
    """T/conftest.py:7-14: every test starts with an empty autotune cache."""
    kernels._autotune_cache.clear()
    yield
    kernels._autotune_cache.clear()


def worst_rel(got, want, floor=1e-6):
    """T/conftest.py:17-22: max |got - want| / max(|want|, floor)."""
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), floor))) if got.size else 0.0


def central_diff(f, x, h_rel=1e-6):
    """F/oracle.py:29-48: element-wise central differences in float64,
    h_i = h_rel * max(1, |x_i|)."""
    x = np.array(x, dtype=np.float64)
    g = np.zeros_like(x)
    fx, fg = x.reshape(-1), g.reshape(-1)
    for i in range(fx.size):
        h = h_rel * max(1.0, abs(fx[i]))
        keep = fx[i]
        fx[i] = keep + h
        up = f(x)
        fx[i] = keep - h
        down = f(x)
        fx[i] = keep
        fg[i] = (up - down) / (2.0 * h)
    return g


def fd_err(analytic, f, x):
    """F/gradcheck.py:19,51: worst relative error against FD, floor 1e-6."""
    return worst_rel(analytic, central_diff(f, x), floor=1e-6)


# ======================================================================
# T/test_kernels.py
# ======================================================================

# --- layernorm (T/test_kernels.py:19-66) --------------------------------

def test_layernorm_two_point_row_is_its_own_normalisation():          # :19-22
    y, cache = K.layernorm_forward(np.array([[1.0, -1.0]]), np.ones(2), np.zeros(2), eps=0.0)
    assert np.allclose(y, [[1.0, -1.0]])
    assert cache.mu[0] == 0.0 and cache.sigma[0] == 1.0


def test_layernorm_of_constant_rows_is_the_bias():                    # :25-30
    b = np.array([0.5, -1.0, 2.0, 0.0])
    y, _ = K.layernorm_forward(np.full((3, 4), 2.5), np.arange(1.0, 5.0), b, eps=1e-5)
    assert np.allclose(y, np.broadcast_to(b, (3, 4)))


def test_layernorm_known_row_1234():                                  # :33-41
    x = np.array([[1.0, 2.0, 3.0, 4.0]])
    want = (x - 2.5) / math.sqrt(1.25)
    y, cache = K.layernorm_forward(x, np.ones(4), np.zeros(4), eps=0.0)
    assert np.allclose(y, want, atol=1e-12)
    assert cache.sigma[0] == pytest.approx(math.sqrt(1.25), abs=1e-12)
    assert np.allclose(y, [[-1.34164, -0.44721, 0.44721, 1.34164]], atol=1e-5)


def test_layernorm_zero_variance_without_eps_raises():                # :44-46
    with pytest.raises(DegenerateRow):
        K.layernorm_forward(np.full((1, 4), 3.0), np.ones(4), np.zeros(4), eps=0.0)


@given(arrays(np.float64, (3, 8), elements=st.floats(-100, 100)))
@FEW
def test_layernorm_output_has_zero_mean_unit_variance(x):             # :49-55
    x = x + np.arange(8) * 1e-3
    y, _ = K.layernorm_forward(x, np.ones(8), np.zeros(8), eps=0.0)
    assert np.abs(y.mean(axis=-1)).max() < 1e-6
    assert np.abs(np.square(y).mean(axis=-1) - 1.0).max() < 1e-5


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_single_pass_sigma_survives_a_large_shift(dtype):             # :58-64
    x = (np.random.default_rng(0).normal(0, 1, (64, 16)) + 1000.0).astype(dtype)
    _, cache = K.layernorm_forward(x, np.ones(16, dtype), np.zeros(16, dtype), eps=0.0)
    xd = x.astype(np.float64)
    two_pass = np.sqrt(np.square(xd - xd.mean(axis=1, keepdims=True)).mean(axis=1))
    assert worst_rel(cache.sigma, two_pass) < 1e-5


# --- softmax family (T/test_kernels.py:69-140) ---------------------------

def test_softmax_equal_logits_are_uniform():                          # :69-72
    y, cache = K.softmax_forward(np.array([[3.0, 3.0, 3.0]]))
    assert np.allclose(y, 1.0 / 3.0)
    assert cache.probs is y


def test_softmax_single_kept_position_gets_all_mass():                # :75-78
    y, _ = K.softmax_forward(np.array([[1.0, 1.0]]), mask=np.array([[True, False]]))
    assert np.array_equal(y, [[1.0, 0.0]])


def test_softmax_known_row_123():                                     # :81-87
    x = np.array([1.0, 2.0, 3.0])
    e = np.exp(x - 3.0)
    y, _ = K.softmax_forward(x[None, :])
    assert np.allclose(y[0], e / e.sum(), atol=1e-12)
    assert np.allclose(y[0], [0.0900306, 0.2447285, 0.6652410], atol=1e-6)


def test_softmax_row_without_kept_positions_raises():                 # :90-92
    with pytest.raises(AllMaskedRow):
        K.softmax_forward(np.ones((1, 3)), mask=np.zeros((1, 3), dtype=bool))


def test_softmax_f32_rows_sum_to_one():                               # :95-99
    x = np.random.default_rng(1).normal(0, 5, (50, 17)).astype(np.float32)
    y, _ = K.softmax_forward(x)
    assert y.dtype == np.float32
    assert np.abs(y.sum(axis=-1) - 1.0).max() < 1e-6


@given(arrays(np.int64, (4, 9), elements=st.integers(-800, 800)), st.integers(-480, 480))
@FEW
def test_softmax_exact_shift_moves_nothing_beyond_one_ulp(xi, ci):    # :102-114
    x = (xi / 16.0).astype(np.float32)        # dyadic: x + c is exact in binary32
    c = np.float32(ci / 16.0)
    a, _ = K.softmax_forward(x)
    b, _ = K.softmax_forward(x + c)
    ulp = np.spacing(np.maximum(np.abs(a), np.abs(b)).astype(np.float32))
    assert np.all(np.abs(a - b) <= ulp)


def test_log_softmax_uniform_and_dominant_logit():                    # :117-122
    assert np.allclose(K.log_softmax_forward(np.array([[0.0, 0.0]])), -math.log(2.0))
    y = K.log_softmax_forward(np.array([[1000.0, 0.0]]))
    assert np.all(np.isfinite(y)) and np.allclose(y, [[0.0, -1000.0]], atol=1e-9)


def test_log_softmax_known_row_123():                                 # :125-131
    h = np.array([[1.0, 2.0, 3.0]])
    want = (h - 3.0) - np.log(np.exp(h - 3.0).sum())
    y = K.log_softmax_forward(h)
    assert np.allclose(y, want, atol=1e-12)
    assert np.allclose(y, [[-2.40761, -1.40761, -0.40761]], atol=1e-5)


def test_log_softmax_stays_finite_for_logits_up_to_1e4():             # :134-138
    h = np.random.default_rng(2).uniform(-1e4, 1e4, (20, 33))
    assert np.all(np.isfinite(K.log_softmax_forward(h)))


# --- reduction strategies (T/test_kernels.py:143-171) --------------------

def test_strategy_rule_by_row_width():                                # :143-147
    assert K.select_softmax_strategy(10**6, 8) == K.ROW_SERIAL
    assert K.select_softmax_strategy(4, 10**5) == K.ROW_PARALLEL_TREE
    assert K.select_softmax_strategy(7, 4096) == K.ROW_SERIAL
    assert K.select_softmax_strategy(7, 4097) == K.ROW_PARALLEL_TREE


def test_autotuned_strategy_is_cached_and_reused():                   # :150-157
    first = K.select_softmax_strategy(64, 333, autotune=True)
    assert (64, 333) in kernels._autotune_cache
    assert first in (K.ROW_SERIAL, K.ROW_PARALLEL_TREE)
    assert K.select_softmax_strategy(64, 333, autotune=True) == first
    assert K.select_softmax_strategy(64, 333) == first     # honoured without the flag


@pytest.mark.parametrize("shape", [(5, 3), (7, 64), (3, 100), (2, 1000), (4, 512), (3, 1024)])
def test_serial_and_tree_strategies_agree_to_one_ulp(shape):          # :160-171
    x = np.random.default_rng(42).normal(0, 10, shape).astype(np.float32)
    a, _ = K.softmax_forward(x, strategy=K.ROW_SERIAL)
    b, _ = K.softmax_forward(x, strategy=K.ROW_PARALLEL_TREE)
    assert np.all(np.abs(a - b) <= np.spacing(np.abs(a).astype(np.float32)))
    la = K.log_softmax_forward(x, strategy=K.ROW_SERIAL)
    lb = K.log_softmax_forward(x, strategy=K.ROW_PARALLEL_TREE)
    assert np.all(np.abs(la - lb) <= np.spacing(np.maximum(np.abs(la), 1.0).astype(np.float32)))
    # and both sit on the float64 softmax within the 1e-6 of T/test_kernels.py:359-374
    assert worst_rel(a, O.softmax_fwd(x.astype(np.float64)), floor=1.0) < 1e-6


def test_strategies_agree_under_masks():
    """Both strategies honour dense / causal / padding masks identically."""
    rng = np.random.default_rng(5)
    x = rng.normal(0, 3, (2, 3, 16, 16)).astype(np.float32)
    for mask in (AttentionMask("causal"), AttentionMask("padding", np.array([5, 16])),
                 rng.random((2, 3, 16, 16)) > 0.3):
        if isinstance(mask, np.ndarray):
            mask[..., 0] = True
        a, _ = K.softmax_forward(x, mask=mask, strategy=K.ROW_SERIAL)
        b, _ = K.softmax_forward(x, mask=mask, strategy=K.ROW_PARALLEL_TREE)
        assert np.all(np.abs(a - b) <= np.spacing(np.abs(a).astype(np.float32)))


# --- criterion (T/test_kernels.py:176-208) --------------------------------

def test_plain_cross_entropy_of_a_fair_coin_is_ln2():                 # :176-180
    loss, count = K.ls_cross_entropy_forward(np.log(np.full((1, 2), 0.5)), [0], alpha=0.0)
    assert loss == pytest.approx(math.log(2.0), rel=1e-12) and count == 1


@pytest.mark.parametrize("v", [2, 5, 32])
def test_fully_smoothed_uniform_prediction_costs_ln_v(v):             # :183-187
    loss, _ = K.ls_cross_entropy_forward(np.full((1, v), -math.log(v)), [1], alpha=1.0)
    assert loss == pytest.approx(math.log(v), rel=1e-12)


@pytest.mark.parametrize("alpha", [0.0, 0.1, 0.5, 1.0])
def test_uniform_prediction_loss_does_not_depend_on_alpha(alpha):     # :190-194
    logq = K.log_softmax_forward(np.zeros((1, 4)))
    loss, _ = K.ls_cross_entropy_forward(logq, [0], alpha=alpha)
    assert loss == pytest.approx(math.log(4.0), rel=1e-12)


def test_pad_targets_are_excluded_and_bad_targets_raise():            # :197-202
    logq = K.log_softmax_forward(np.zeros((3, 4)))
    loss, count = K.ls_cross_entropy_forward(logq, [0, 1, 0], alpha=0.0, pad_id=0)
    assert count == 1 and loss == pytest.approx(math.log(4.0), rel=1e-12)
    with pytest.raises(TokenOutOfRange):
        K.ls_cross_entropy_forward(logq, [0, 9, 0], alpha=0.0)


# --- embedding (T/test_kernels.py:205-246) --------------------------------

E2 = np.array([[1.0, 2.0], [3.0, 4.0]])
P2 = np.array([[0.1, 0.2], [0.3, 0.4]])


def test_embedding_is_row_plus_position():                            # :213-218
    y, mask = K.embedding_forward(E2, P2, [[1, 0]], EmbeddingConfig(1.0, 2, 2), 0.0, seed=0)
    assert np.allclose(y[0], [[3.1, 4.2], [1.3, 2.4]]) and np.all(mask.keep == 1)


def test_embedding_scale_multiplies_the_row_only():                   # :221-225
    y, _ = K.embedding_forward(E2, P2, [[1, 0]], EmbeddingConfig(2.0, 2, 2), 0.0, seed=0)
    assert np.allclose(y[0], [[6.1, 8.2], [2.3, 4.4]])


def test_embedding_dropout_follows_the_counter_rng():                 # :228-235
    y, mask = K.embedding_forward(E2, P2, [[1, 0]], EmbeddingConfig(1.0, 2, 2), 0.5, seed=77)
    keep = (host(_numerics.rand_uniform_array(77, 0, 4)) >= 0.5).reshape(1, 2, 2)
    assert np.array_equal(keep, O.counter_uniform(77, 0, 4).reshape(1, 2, 2) >= 0.5)
    assert np.array_equal(mask.keep, keep.astype(mask.keep.dtype))
    assert np.allclose(y, keep * np.array([[[3.1, 4.2], [1.3, 2.4]]]) * 2.0)


def test_embedding_rejects_bad_tokens_and_long_sequences():           # :238-244
    cfg = EmbeddingConfig(1.0, 2, 2)
    with pytest.raises(TokenOutOfRange):
        K.embedding_forward(E2, P2, [[2, 0]], cfg, 0.0, seed=0)
    with pytest.raises(SequenceTooLong):
        K.embedding_forward(E2, P2, [[0, 1, 0]], cfg, 0.0, seed=0)


# --- fused tails (T/test_kernels.py:249-288) ------------------------------

def test_bias_dropout_residual_without_dropout_is_a_sum():            # :249-255
    rng = np.random.default_rng(3)
    x, res, bias = rng.normal(size=(2, 3, 4)), rng.normal(size=(2, 3, 4)), rng.normal(size=4)
    y, mask = K.bias_dropout_residual(x, bias, res, 0.0, seed=0)
    assert np.allclose(y, x + bias + res) and np.all(mask.keep == 1)


@pytest.mark.parametrize("p,seed", [(0.0, 0), (0.5, 9), (0.9, 17)])
def test_bias_dropout_residual_of_a_zero_branch_is_the_residual(p, seed):  # :258-262
    res = np.random.default_rng(4).normal(size=(2, 5))
    y, _ = K.bias_dropout_residual(np.zeros((2, 5)), np.zeros(5), res, p, seed)
    assert np.allclose(y, res)


def test_bias_dropout_residual_equals_the_unfused_chain():            # :265-271
    rng = np.random.default_rng(5)
    x, res, bias = rng.normal(size=(3, 4)), rng.normal(size=(3, 4)), rng.normal(size=4)
    y, mask = K.bias_dropout_residual(x, bias, res, 0.5, seed=21)
    assert worst_rel(y, (x + bias) * mask.keep / 0.5 + res) < 1e-12


def test_bias_relu_dropout_known_values():                            # :274-279
    y, _, relum = K.bias_relu_dropout(np.array([[-1.0, 2.0]]), np.zeros(2), 0.0, seed=0)
    assert np.allclose(y, [[0.0, 2.0]]) and np.array_equal(relum, [[0.0, 1.0]])
    y, _, _ = K.bias_relu_dropout(np.full((2, 3), -4.0), np.ones(3), 0.3, seed=5)
    assert np.all(y == 0.0)


def test_bias_relu_dropout_equals_the_unfused_chain():                # :282-288
    rng = np.random.default_rng(6)
    x, bias = rng.normal(size=(4, 6)), rng.normal(size=6)
    y, mask, _ = K.bias_relu_dropout(x, bias, 0.5, seed=33)
    assert worst_rel(y, np.maximum(x + bias, 0.0) * mask.keep / 0.5) < 1e-12


# --- gemm (T/test_kernels.py:293-320) -------------------------------------

def test_gemm_identity_and_a_small_known_product():                   # :293-297
    a = np.random.default_rng(7).normal(size=(3, 3))
    assert np.allclose(K.gemm(a, np.eye(3)), a)
    c = K.gemm(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0, 6.0], [7.0, 8.0]]))
    assert np.array_equal(c, [[19.0, 22.0], [43.0, 50.0]])


def test_gemm_transpose_flags():                                      # :300-305
    rng = np.random.default_rng(8)
    a, b = rng.normal(size=(4, 3)), rng.normal(size=(4, 5))
    assert np.allclose(K.gemm(a, b, trans_a=True), a.T @ b)
    x, y = rng.normal(size=(5, 3)), rng.normal(size=(4, 3))
    assert np.allclose(K.gemm(x, y, trans_b=True), x @ y.T)


def test_gemm_shape_error_and_in_place_accumulation():                # :308-313
    with pytest.raises(ShapeMismatch):
        K.gemm(np.zeros((2, 3)), np.zeros((4, 2)))
    acc = np.ones((2, 2))
    K.gemm(np.eye(2), np.eye(2), accumulate_into=acc)
    assert np.array_equal(acc, np.eye(2) + 1.0)


def test_gemm_long_reduction_matches_the_direct_product():            # :316-320
    rng = np.random.default_rng(9)
    k = 2 * K.GEMM_BLOCK_K + 17
    a, b = rng.normal(size=(3, k)), rng.normal(size=(k, 4))
    assert worst_rel(K.gemm(a, b), a @ b) < 1e-12


# --- masks, dtypes, determinism (T/test_kernels.py:325-374) ---------------

def test_attention_mask_kinds_materialise():                          # :325-333
    assert AttentionMask("none").keep_array(3, 3) is None
    assert np.array_equal(host(AttentionMask("causal").keep_array(3, 3)),
                          np.tril(np.ones((3, 3), bool)))
    padk = host(AttentionMask("padding", np.array([2, 3])).keep_array(4, 3))
    assert padk.shape == (2, 1, 1, 3) and np.array_equal(padk[0, 0, 0], [True, True, False])
    with pytest.raises(ShapeMismatch):
        AttentionMask("padding", np.array([0])).keep_array(2, 2)


def test_fused_forward_ops_are_bitwise_repeatable():                  # :336-348
    """The reference pins thread-count invariance; the device analogue is that
    two launches (no CPU pool) return identical bits."""
    x = np.random.default_rng(10).normal(size=(4096, 32)).astype(np.float32)
    w, b = np.ones(32, np.float32), np.zeros(32, np.float32)
    y1, _ = K.softmax_forward(x)
    l1, c1 = K.layernorm_forward(x, w, b, 1e-5)
    y3, _ = K.softmax_forward(x)
    l3, c3 = K.layernorm_forward(x, w, b, 1e-5)
    assert np.array_equal(y1, y3) and np.array_equal(l1, l3)
    assert np.array_equal(c1.sigma, c3.sigma)


def test_float16_inputs_give_float32_outputs():                      # :351-356
    x = np.random.default_rng(11).normal(size=(3, 8)).astype(np.float16)
    y, _ = K.layernorm_forward(x, np.ones(8, np.float16), np.zeros(8, np.float16), 1e-5)
    s, _ = K.softmax_forward(x)
    assert y.dtype == np.float32 and s.dtype == np.float32


def test_binary32_fused_ops_sit_within_1e6_of_float64():              # :359-374
    rng = np.random.default_rng(12)
    x = rng.normal(size=(6, 16)).astype(np.float32)
    w, b = rng.normal(size=16).astype(np.float32), rng.normal(size=16).astype(np.float32)
    y, _ = K.layernorm_forward(x, w, b, 1e-5)
    want, _, _ = O.layernorm_fwd(x.astype(np.float64), w.astype(np.float64), b.astype(np.float64))
    assert worst_rel(y, want, floor=1.0) < 1e-6
    s, _ = K.softmax_forward(x)
    assert worst_rel(s, O.softmax_fwd(x.astype(np.float64)), floor=1.0) < 1e-6
    res = rng.normal(size=(6, 16)).astype(np.float32)
    yf, mask = K.bias_dropout_residual(x, b, res, 0.5, seed=6)
    ref = (x.astype(np.float64) + b) * mask.keep / 0.5 + res
    assert worst_rel(yf, ref, floor=1.0) < 1e-6


# ======================================================================
# T/test_gradients.py
# ======================================================================

def test_embedding_backward_sums_a_repeated_token():                  # :16-24
    cfg = EmbeddingConfig(scale=2.0, vocab=8, max_len=4)
    dy = np.arange(8.0).reshape(1, 2, 4)
    de, dp = G.embedding_backward(dy, [[5, 5]], DropoutMask(np.ones((1, 2, 4)), 0.0), cfg)
    assert np.allclose(de[5], 2.0 * (dy[0, 0] + dy[0, 1]))
    assert np.all(np.delete(de, 5, axis=0) == 0.0)
    assert np.allclose(dp[:2], dy[0])


def test_embedding_backward_through_an_all_drop_mask_is_zero():       # :27-31
    cfg = EmbeddingConfig(scale=1.0, vocab=4, max_len=3)
    de, dp = G.embedding_backward(np.ones((1, 3, 2)), [[0, 1, 2]],
                                  DropoutMask(np.zeros((1, 3, 2)), 0.5), cfg)
    assert np.all(de == 0.0) and np.all(dp == 0.0)


@pytest.mark.parametrize("i", range(5))
def test_embedding_backward_matches_finite_differences(i):            # :34-35, F/gradcheck.py:33-55
    rng = np.random.default_rng(i)
    v, b, l, d = 7, 2, 3, 4
    cfg = EmbeddingConfig(scale=1.5, vocab=v, max_len=l)
    emb, pos = rng.normal(size=(v, d)), rng.normal(size=(l, d))
    tokens, w = rng.integers(0, v, (b, l)), rng.normal(size=(b, l, d))
    p, seed = (0.5 if i % 2 else 0.0), 17 + i

    def f(e, tab):
        return float((w * K.embedding_forward(e, tab, tokens, cfg, p, seed)[0]).sum())

    _, mask = K.embedding_forward(emb, pos, tokens, cfg, p, seed)
    de, dp = G.embedding_backward(w, tokens, mask, cfg)
    assert fd_err(de, lambda e: f(e, pos), emb) < 1e-5
    assert fd_err(dp, lambda t: f(emb, t), pos) < 1e-5


def test_embedding_gradient_mass_is_conserved():                      # :38-47
    rng = np.random.default_rng(0)
    cfg = EmbeddingConfig(scale=1.7, vocab=9, max_len=5)
    tokens, dy = rng.integers(0, 9, (2, 5)), rng.normal(size=(2, 5, 3))
    _, mask = K.embedding_forward(rng.normal(size=(9, 3)), rng.normal(size=(5, 3)), tokens,
                                  cfg, 0.5, seed=3)
    de, _ = G.embedding_backward(dy, tokens, mask, cfg)
    assert worst_rel(de.sum(axis=0), 1.7 * (mask.keep * dy / 0.5).reshape(-1, 3).sum(axis=0)) < 1e-6


def test_ce_backward_fair_coin():                                     # :52-54
    assert np.allclose(G.ls_cross_entropy_backward(np.array([[0.5, 0.5]]), [0], alpha=0.0),
                       [[-0.5, 0.5]])


def test_ce_backward_smoothed_uniform_row():                          # :57-61
    dh = G.ls_cross_entropy_backward(np.full((1, 4), 0.25), [0], alpha=0.1)
    assert np.allclose(dh, [[-0.675, 0.225, 0.225, 0.225]], atol=1e-12)
    assert abs(dh.sum()) < 1e-12


@given(arrays(np.float64, (3, 6), elements=st.floats(-5, 5)), st.floats(0, 1))
@FEW
def test_ce_backward_rows_sum_to_zero(h, alpha):                      # :64-70
    q, _ = K.softmax_forward(h)
    dh = G.ls_cross_entropy_backward(q, np.array([0, 3, 5]), alpha=alpha)
    assert np.abs(dh.sum(axis=-1)).max() < 1e-12


def test_ce_backward_pad_rows_are_zero():                             # :73-76
    dh = G.ls_cross_entropy_backward(np.full((2, 4), 0.25), [0, 2], alpha=0.0, pad_id=0)
    assert np.all(dh[0] == 0.0) and not np.all(dh[1] == 0.0)


@pytest.mark.parametrize("i", range(6))
def test_ce_backward_matches_finite_differences(i):                   # :79-80, F/gradcheck.py:58-76
    rng = np.random.default_rng(1000 + i)
    h = rng.normal(size=(3, 6)) * 2.0
    targets = rng.integers(0, 6, 3)
    targets[0] = 0
    alpha = [0.0, 0.1, 1.0][i % 3]

    def f(x):
        return K.ls_cross_entropy_forward(K.log_softmax_forward(x), targets, alpha, pad_id=0)[0]

    probs, _ = K.softmax_forward(h)
    assert fd_err(G.ls_cross_entropy_backward(probs, targets, alpha, pad_id=0), f, h) < 1e-5


def test_softmax_backward_annihilates_a_constant_gradient():          # :85-88
    _, cache = K.softmax_forward(np.random.default_rng(1).normal(size=(2, 5)))
    assert np.abs(G.softmax_backward(np.full((2, 5), 3.3), cache)).max() < 1e-12


def test_softmax_backward_of_a_saturated_row_is_zero():               # :91-94
    dx = G.softmax_backward(np.array([[2.0, -1.0, 0.5]]), SoftmaxCache(np.array([[1.0, 0.0, 0.0]])))
    assert np.abs(dx).max() < 1e-12


@pytest.mark.parametrize("i", range(10))
def test_softmax_backward_matches_finite_differences(i):              # :97-99, F/gradcheck.py:79-94
    rng = np.random.default_rng(2000 + i)
    x, w = rng.normal(size=(3, 5)) * 2.0, rng.normal(size=(3, 5))
    _, cache = K.softmax_forward(x)
    dx = G.softmax_backward(w, cache)
    assert fd_err(dx, lambda t: float((w * K.softmax_forward(t)[0]).sum()), x) < 1e-5


def test_softmax_backward_random_row_within_1e6_of_fd():             # :102-119
    rng = np.random.default_rng(7)
    x, w = rng.normal(size=(1, 5)) * 2.0, rng.normal(size=(1, 5))
    _, cache = K.softmax_forward(x)
    dx = G.softmax_backward(w, cache)
    fd = central_diff(lambda t: float((w * K.softmax_forward(t)[0]).sum()), x)
    assert np.abs(dx - fd).max() <= 1e-6 * max(1.0, np.abs(fd).max())


@given(arrays(np.float64, (2, 8), elements=st.floats(-50, 50)),
       arrays(np.float64, (8,), elements=st.floats(-2, 2)),
       arrays(np.float64, (2, 8), elements=st.floats(-3, 3)))
@FEW
def test_layernorm_backward_rows_sum_to_zero(x, w, dy):               # :122-129
    x = x + np.arange(8.0) * 0.1
    _, cache = K.layernorm_forward(x, w, np.zeros(8), eps=1e-5)
    dx, _, _ = G.layernorm_backward(dy, x, w, cache)
    assert np.abs(dx.sum(axis=-1)).max() < 1e-10


def _textbook_ln_backward(dy, x, w, mu, sigma):
    """Direct LayerNorm backward: dx = (g - mean(g) - xhat*mean(g*xhat)) / sigma."""
    xhat = (x - mu[:, None]) / sigma[:, None]
    g = w * dy
    dx = (g - g.mean(axis=1, keepdims=True)
          - xhat * (g * xhat).mean(axis=1, keepdims=True)) / sigma[:, None]
    return dx, (dy * xhat).sum(axis=0), dy.sum(axis=0)


def test_layernorm_backward_kills_the_normalised_direction():         # :132-142
    x = np.random.default_rng(2).normal(size=(4, 8)) * 2
    _, cache = K.layernorm_forward(x, np.ones(8), np.zeros(8), eps=0.0)
    xhat = (x - cache.mu[:, None]) / cache.sigma[:, None]
    dx, _, _ = G.layernorm_backward(xhat, x, np.ones(8), cache)
    assert np.abs(dx).max() < 1e-8
    assert np.abs(_textbook_ln_backward(xhat, x, np.ones(8), cache.mu, cache.sigma)[0]).max() < 1e-8


def test_layernorm_rearranged_backward_equals_the_textbook_form():    # :145-157
    rng = np.random.default_rng(3)
    for _ in range(50):
        m = int(rng.integers(2, 17))
        x = rng.normal(size=(3, m)) * rng.uniform(0.1, 10)
        w, dy = rng.normal(size=m), rng.normal(size=(3, m))
        _, cache = K.layernorm_forward(x, w, np.zeros(m), eps=1e-5)
        dx, dw, db = G.layernorm_backward(dy, x, w, cache)
        dxt, dwt, dbt = _textbook_ln_backward(dy, x, w, cache.mu, cache.sigma)
        assert np.abs(dx - dxt).max() < 1e-12 * max(1.0, np.abs(dxt).max())
        assert np.allclose(dw, dwt, atol=1e-10) and np.allclose(db, dbt, atol=1e-10)


@pytest.mark.parametrize("i", range(10))
def test_layernorm_backward_matches_finite_differences(i):            # :160-161, F/gradcheck.py:97-118
    rng = np.random.default_rng(3000 + i)
    x = rng.normal(size=(2, 8)) * 3.0
    w, b, dy = rng.normal(size=8), rng.normal(size=8), rng.normal(size=(2, 8))

    def f(t, wt=w, bt=b):
        return float((dy * K.layernorm_forward(t, wt, bt, 1e-5)[0]).sum())

    _, cache = K.layernorm_forward(x, w, b, 1e-5)
    dx, dw, db = G.layernorm_backward(dy, x, w, cache)
    assert fd_err(dx, f, x) < 1e-5
    assert fd_err(dw, lambda t: f(x, wt=t), w) < 1e-5
    assert fd_err(db, lambda t: f(x, bt=t), b) < 1e-5


def test_bias_dropout_residual_backward_without_dropout():           # :166-172
    dy = np.random.default_rng(4).normal(size=(2, 3, 4))
    dx, dbias, dres = G.bias_dropout_residual_backward(dy, DropoutMask(np.ones((2, 3, 4)), 0.0))
    assert np.array_equal(dx, dy) and np.array_equal(dres, dy)
    assert np.allclose(dbias, dy.reshape(-1, 4).sum(axis=0))


def test_bias_dropout_residual_backward_through_an_all_drop_mask():  # :175-180
    dy = np.ones((2, 4))
    dx, dbias, dres = G.bias_dropout_residual_backward(dy, DropoutMask(np.zeros((2, 4)), 0.3))
    assert np.all(dx == 0.0) and np.all(dbias == 0.0) and np.array_equal(dres, dy)


@pytest.mark.parametrize("i", range(6))
def test_bias_dropout_residual_backward_matches_fd(i):                # :183-184, F/gradcheck.py:121-143
    rng = np.random.default_rng(4000 + i)
    x, bias = rng.normal(size=(2, 3, 4)), rng.normal(size=4)
    res, w = rng.normal(size=(2, 3, 4)), rng.normal(size=(2, 3, 4))
    p, seed = (0.4 if i % 2 else 0.0), 23 + i

    def f(t, bt=bias, rt=res):
        return float((w * K.bias_dropout_residual(t, bt, rt, p, seed)[0]).sum())

    _, mask = K.bias_dropout_residual(x, bias, res, p, seed)
    dx, dbias, dres = G.bias_dropout_residual_backward(w, mask)
    assert fd_err(dx, f, x) < 1e-5
    assert fd_err(dbias, lambda t: f(x, bt=t), bias) < 1e-5
    assert fd_err(dres, lambda t: f(x, rt=t), res) < 1e-5


def test_bias_relu_dropout_backward_gates():                          # :187-193
    dy = np.random.default_rng(5).normal(size=(3, 4))
    ones = DropoutMask(np.ones((3, 4)), 0.0)
    dx, _ = G.bias_relu_dropout_backward(dy, ones, np.ones((3, 4)))
    assert np.array_equal(dx, dy)
    dx, dbias = G.bias_relu_dropout_backward(dy, ones, np.zeros((3, 4)))
    assert np.all(dx == 0.0) and np.all(dbias == 0.0)


@pytest.mark.parametrize("i", range(6))
def test_bias_relu_dropout_backward_matches_fd(i):                    # :196-197, F/gradcheck.py:146-171
    rng = np.random.default_rng(5000 + i)
    x, bias = rng.normal(size=(2, 3, 4)), rng.normal(size=4)
    pre = x + bias
    x = x + np.where(np.abs(pre) < 1e-3, np.sign(pre + 1e-12) * 2e-3, 0.0)   # off the kink
    w = rng.normal(size=(2, 3, 4))
    p, seed = (0.4 if i % 2 else 0.0), 29 + i

    def f(t, bt=bias):
        return float((w * K.bias_relu_dropout(t, bt, p, seed)[0]).sum())

    _, mask, relum = K.bias_relu_dropout(x, bias, p, seed)
    dx, dbias = G.bias_relu_dropout_backward(w, mask, relum)
    assert fd_err(dx, f, x) < 1e-5
    assert fd_err(dbias, lambda t: f(x, bt=t), bias) < 1e-5


def test_layernorm_backward_is_bitwise_repeatable():                  # :200-212
    rng = np.random.default_rng(6)
    x, dy, w = rng.normal(size=(4096, 16)), rng.normal(size=(4096, 16)), rng.normal(size=16)
    _, cache = K.layernorm_forward(x, w, np.zeros(16), 1e-5)
    a = G.layernorm_backward(dy, x, w, cache)
    b = G.layernorm_backward(dy, x, w, cache)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


# ======================================================================
# T/test_trainer.py
# ======================================================================

def _rne(x):
    return np.asarray(x, np.float32).astype(np.float16)


def _pack(seed=0, sizes=((3, 2), (4,)), algorithm="adam"):
    rng = np.random.default_rng(seed)
    named = [(f"p{i}", rng.normal(size=s).astype(np.float32)) for i, s in enumerate(sizes)]
    return named, T.workspace_pack(named, algorithm)


def _bits(t):
    return host(t).view(np.uint16)


def test_pack_concatenates_in_order_with_links():                     # :19-27
    a, b = np.arange(6.0, dtype=np.float32).reshape(2, 3), np.arange(4.0, dtype=np.float32)
    ws = T.workspace_pack([("A", a), ("B", b)])
    assert ws.params16.numel() == 10
    assert [(lk.name, lk.offset, lk.length) for lk in ws.links] == [("A", 0, 6), ("B", 6, 4)]
    assert ws.resolve("B") == (6, 4)
    assert np.array_equal(host(ws.param_view("A")), _rne(a))
    assert ws.param_view("B").untyped_storage().data_ptr() == ws.params16.untyped_storage().data_ptr()


def test_packed_values_are_the_rne_of_the_originals():                # :30-34
    x = np.random.default_rng(1).normal(size=17).astype(np.float32) * 3.3
    assert np.array_equal(host(T.workspace_pack([("x", x)]).param_view("x")), x.astype(np.float16))


def test_links_tile_the_workspace_without_gaps():                     # :37-44
    _, ws = _pack(sizes=((3, 2), (4,), (2, 2, 2)))
    pos = 0
    for off, length in sorted((lk.offset, lk.length) for lk in ws.links):
        assert off == pos
        pos += length
    assert pos == ws.params16.numel()


def test_duplicate_parameter_name_raises():                           # :47-49
    with pytest.raises(DuplicateName):
        T.workspace_pack([("x", np.zeros(2)), ("x", np.zeros(3))])


def test_zero_grads_writes_positive_zero_and_leaves_params():        # :52-61
    _, ws = _pack()
    ws.grads16.fill_(1.5)
    before = _bits(ws.params16).copy()
    T.zero_grads(ws)
    assert np.all(_bits(ws.grads16) == 0)
    T.zero_grads(ws)
    assert np.all(_bits(ws.grads16) == 0) and np.array_equal(_bits(ws.params16), before)


@pytest.mark.parametrize("kw", [dict(lr=0.0), dict(beta1=1.0), dict(loss_scale=3.0),
                                dict(loss_scale=0.5)])
def test_optim_config_rejects_bad_values(kw):                         # :64-75
    with pytest.raises(ConfigError):
        T.OptimConfig(**kw)


def test_optim_config_accepts_a_large_power_of_two_scale():           # :75
    T.OptimConfig(loss_scale=65536.0)


def test_adam_with_zero_gradient_changes_nothing():                   # :78-85
    _, ws = _pack()
    before = _bits(ws.params16).copy()
    assert T.adam_step(ws, T.OptimConfig(lr=0.01), t=1).applied
    assert np.array_equal(_bits(ws.params16), before)
    assert not host(ws.m32).any() and not host(ws.v32).any()


def test_adam_scalar_known_value():                                   # :88-97
    ws = T.workspace_pack([("p", np.array([1.0], dtype=np.float32))])
    ws.grads16.fill_(0.1)
    T.adam_step(ws, T.OptimConfig(lr=0.01, beta1=0.9, beta2=0.999, eps_opt=1e-8), t=1)
    g = float(np.float16(0.1))
    want = 1.0 - 0.01 * (g / (abs(g) + 1e-8))
    assert abs(want - 0.99) < 1e-4 and abs(float(host(ws.params16)[0]) - want) < 5e-4


def test_adam_is_bit_exact_against_the_reference_update():            # :100-129
    rng = np.random.default_rng(2)
    for trial in range(50):
        n = int(rng.integers(1, 33))
        p0 = (rng.normal(size=n) * rng.choice([0.01, 1.0, 30.0])).astype(np.float32)
        g0 = (rng.normal(size=n) * rng.choice([1e-4, 0.1, 5.0])).astype(np.float32)
        m0 = rng.normal(size=n).astype(np.float32) * 0.1
        v0 = rng.uniform(0.0, 0.2, size=n).astype(np.float32)
        lr, wd = float(rng.choice([1e-4, 1e-3, 0.01])), float(rng.choice([0.0, 0.01]))
        t, scale = int(rng.integers(1, 50)), float(rng.choice([1.0, 8.0]))
        cfg = T.OptimConfig(lr=lr, weight_decay=wd, loss_scale=scale)
        ws = T.workspace_pack([("p", p0)])
        ws.grads16.copy_(torch.from_numpy(_rne(g0)))
        ws.m32.copy_(torch.from_numpy(m0))
        ws.v32.copy_(torch.from_numpy(v0))
        T.adam_step(ws, cfg, t=t)
        p, m, v = _rne(p0), m0.copy(), v0.copy()
        assert O.adam_flat(p, _rne(g0), m, v, lr=lr, beta1=cfg.beta1, beta2=cfg.beta2,
                           eps=cfg.eps_opt, wd=wd, loss_scale=scale, t=t) == 0
        assert np.array_equal(_bits(ws.params16), p.view(np.uint16)), trial
        assert np.array_equal(host(ws.m32), m) and np.array_equal(host(ws.v32), v), trial


def test_adam_skips_the_step_on_a_non_finite_gradient():              # :132-144
    _, ws = _pack(seed=3)
    ws.grads16.fill_(0.5)
    ws.grads16[2] = float("inf")
    ws.m32.fill_(0.25)
    p_before, m_before = _bits(ws.params16).copy(), host(ws.m32).copy()
    rep = T.adam_step(ws, T.OptimConfig(), t=1)
    assert not rep.applied and rep.nonfinite == 1
    assert np.array_equal(_bits(ws.params16), p_before) and np.array_equal(host(ws.m32), m_before)


def test_sgd_plain_step():                                            # :147-151
    ws = T.workspace_pack([("p", np.array([1.0], dtype=np.float32))], algorithm="sgd")
    ws.grads16.fill_(0.5)
    T.sgd_step(ws, T.OptimConfig(algorithm="sgd", lr=0.1, momentum=0.0))
    assert float(host(ws.params16)[0]) == pytest.approx(0.95, abs=1e-3)


def test_sgd_with_zero_gradient_changes_nothing():                   # :154-158
    _, ws = _pack(algorithm="sgd")
    before = _bits(ws.params16).copy()
    T.sgd_step(ws, T.OptimConfig(algorithm="sgd", lr=0.1, momentum=0.9))
    assert np.array_equal(_bits(ws.params16), before)


def test_sgd_descends_a_quadratic_bowl_like_float64():                # :161-175
    ws = T.workspace_pack([("x", np.array([2.0], dtype=np.float32))], algorithm="sgd")
    cfg = T.OptimConfig(algorithm="sgd", lr=0.1, momentum=0.9)
    ref_x, ref_v = 2.0, 0.0
    for _ in range(10):
        x = float(host(ws.params16)[0])
        ws.grads16.fill_(float(np.float16(np.float32(x))))
        T.sgd_step(ws, cfg)
        ref_v = 0.9 * ref_v + float(np.float16(ref_x))
        ref_x = ref_x - 0.1 * ref_v
        assert abs(float(host(ws.params16)[0]) - ref_x) < 2e-3
        ref_x = float(np.float16(ref_x))


def test_sgd_is_bit_exact_against_the_reference_update():             # :178-198
    rng = np.random.default_rng(4)
    for trial in range(30):
        n = int(rng.integers(1, 20))
        p0, g0 = rng.normal(size=n).astype(np.float32), rng.normal(size=n).astype(np.float32)
        vel0 = rng.normal(size=n).astype(np.float32) * 0.1
        ws = T.workspace_pack([("p", p0)], algorithm="sgd")
        ws.grads16.copy_(torch.from_numpy(_rne(g0)))
        ws.m32.copy_(torch.from_numpy(vel0))
        T.sgd_step(ws, T.OptimConfig(algorithm="sgd", lr=0.05, momentum=0.9, weight_decay=0.01))
        p, vel = _rne(p0), vel0.copy()
        assert O.sgd_flat(p, _rne(g0), vel, lr=0.05, momentum=0.9, wd=0.01, loss_scale=1.0) == 0
        assert np.array_equal(_bits(ws.params16), p.view(np.uint16)), trial
        assert np.array_equal(host(ws.m32), vel), trial


def test_workspace_state_is_2p_fp16_plus_2p_fp32():                   # :201-207
    _, ws = _pack(seed=5, sizes=((10, 3), (7,), (4, 4)))
    p = ws.n_elements
    assert ws.state_bytes() == 2 * p * 2 + 2 * p * 4
    # the per-tensor fp32-master baseline (F/oracle.py BaselineTrainer) holds 2P more fp32


def test_twenty_adam_steps_stay_bit_exact_per_tensor():               # :210-226
    rng = np.random.default_rng(6)
    named = [("a", rng.normal(size=(4, 3)).astype(np.float32)),
             ("b", rng.normal(size=6).astype(np.float32))]
    cfg = T.OptimConfig(lr=0.01)
    ws = T.workspace_pack(named, "adam")
    ref = {name: [_rne(arr).reshape(-1), np.zeros(arr.size, np.float32),
                  np.zeros(arr.size, np.float32)] for name, arr in named}
    for t in range(1, 21):
        grads = {name: _rne(rng.normal(size=arr.shape) * 0.3) for name, arr in named}
        for name, _ in named:
            ws.grad_view(name).copy_(torch.from_numpy(grads[name]))
        T.adam_step(ws, cfg, t=t)
        for name, _ in named:
            p, m, v = ref[name]
            O.adam_flat(p, grads[name].reshape(-1), m, v, lr=0.01, beta1=0.9, beta2=0.999,
                        eps=1e-8, wd=0.0, loss_scale=1.0, t=t)
            assert np.array_equal(_bits(ws.param_view(name)).reshape(-1), p.view(np.uint16)), (t, name)
