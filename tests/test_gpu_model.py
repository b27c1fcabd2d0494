"""GPU parity of the model composition, workspace step and engine against the
reference's golden vectors (tests/golden/model.npz) and the CPU oracle.

f64: grads within 1e-9 of the reference (the reference's own model-vs-oracle
bar, pkg/tests/test_model.py:228-242); f32: 1e-5 relative; fp16 activations:
2e-2 relative (BASELINE.json north star).
"""

import math

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import lsport as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2110_05722_b200 import model as M
    from paper_2110_05722_b200 import trainer as T
    from paper_2110_05722_b200 import _lib
    from paper_2110_05722_b200.config import RunConfig, TrainConfig
    from paper_2110_05722_b200.engine import TrainingEngine
    from paper_2110_05722_b200.errors import IncompleteGradientSet


def H(t):
    return t.detach().cpu().numpy()


def tiny_golden_cfg():
    return M.ModelConfig(n_enc=2, n_dec=2, d_model=16, n_heads=4, d_ff=24, vocab=19, max_len=8)


def _golden_batch(gm):
    return M.Batch(gm["src"], gm["tgt_in"], gm["tgt_out"], gm["src_len"], 0)


def test_init_params_bit_identical(golden_model):
    cfg = tiny_golden_cfg()
    init = M.init_params(cfg, seed=3)
    for name, _ in M.param_spec(cfg):
        assert np.array_equal(H(init[name]), golden_model[f"init_{name}"]), name


@pytest.mark.parametrize("tag,dt,tol", [("f64", torch.float64, 1e-9), ("f32", torch.float32, 2e-5)])
def test_model_forward_backward_golden(golden_model, tag, dt, tol):
    gm = golden_model
    cfg = tiny_golden_cfg()
    tf = M.Transformer(cfg)
    params = {k: v.to(dt) for k, v in M.init_params(cfg, seed=3).items()}
    sink = M.GradSink()
    cap = {}
    out = tf.forward_backward(params, _golden_batch(gm), p_drop=0.2, alpha=0.1, seed=11, step=4,
                              sink=sink, capture=cap)
    want = gm[f"{tag}_out"]
    assert out.token_count == want[1] and out.correct == want[2]
    assert abs(out.loss_sum - want[0]) <= tol * abs(want[0])
    assert rel_err(H(cap["logq"]), gm[f"{tag}_logq"], 1.0) < tol
    for name, _ in M.param_spec(cfg):
        ref = gm[f"{tag}_g_{name}"]
        got = H(sink.store[name])
        assert np.abs(got - ref).max() <= tol * max(1.0, np.abs(ref).max()), name


def test_view_sink_writes_match_dict_sink(golden_model):
    """Direct workspace writes (_ViewSink) == staged adds (GradSink)."""
    gm = golden_model
    cfg = tiny_golden_cfg()
    tf = M.Transformer(cfg)
    params = {k: v.to(torch.float64) for k, v in M.init_params(cfg, seed=3).items()}
    views = {k: torch.full_like(v, 123.0) for k, v in params.items()}
    tf.forward_backward(params, _golden_batch(gm), p_drop=0.2, alpha=0.1, seed=11, step=4,
                        sink=M._ViewSink(views))
    for name, _ in M.param_spec(cfg):
        ref = gm[f"f64_g_{name}"]
        assert np.abs(H(views[name]) - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max()), name


def test_workspace_engine_steps_vs_reference(golden_model):
    """Engine arithmetic (grad_acc * f32(ls/count) -> narrow -> Adam) on an fp16
    workspace with f32 activations, vs the reference engine's params16."""
    gm = golden_model
    cfg = tiny_golden_cfg()
    tf = M.Transformer(cfg, compute_dtype=torch.float32)
    init = M.init_params(cfg, seed=3)
    ws = T.workspace_pack([(n, init[n]) for n in tf.param_names], "adam")
    pv = ws.param_views()
    acc = torch.zeros(ws.n_elements, device="cuda")
    gv = {lk.name: acc[lk.offset:lk.offset + lk.length].view(lk.shape) for lk in ws.links}
    ocfg = T.OptimConfig(lr=2e-3, loss_scale=4.0)
    for step in range(3):
        out = tf.forward_backward(pv, _golden_batch(gm), p_drop=0.1, alpha=0.1, seed=7, step=step,
                                  sink=M._ViewSink(gv))
        want = gm[f"eng_loss_{step}"]
        assert abs(out.loss_sum - want[0]) <= 1e-5 * abs(want[0])
        _lib.call("ls2_scale_narrow", acc.data_ptr(), ws.grads16.data_ptr(), ws.n_elements, 4.0,
                  out.out3.data_ptr(), -1, 1.0, None, _lib.stream_handle())
        g16 = H(ws.grads16).astype(np.float32)
        ref_g = gm[f"eng_g16_{step}"].astype(np.float32)
        assert np.abs(g16 - ref_g).max() <= 2e-3 * max(1.0, np.abs(ref_g).max())
        T.adam_step(ws, ocfg, step + 1)
        ref = gm[f"eng_p16_{step}"].astype(np.float32)
        mine = H(ws.params16).astype(np.float32)
        assert np.mean(mine != ref) < 2e-2
        assert np.abs(mine - ref).max() <= 2e-2 * max(1.0, np.abs(ref).max())


def _tbase_layer_inputs(b=8, l=64, d=512, seed=0):
    rng = np.random.default_rng(seed)
    return rng.normal(size=(b, l, d)).astype(np.float32), rng.normal(size=(b, l, d)).astype(np.float32)


def test_encoder_layer_fp16_vs_oracle_tbase_dims():
    """Config 1 of BASELINE.json (one encoder layer, B8 x L64, d512, h8, f2048),
    fp16 storage vs the f32 oracle with identical dropout masks (p=0.1)."""
    cfg = M.ModelConfig(n_enc=1, n_dec=1, d_model=512, n_heads=8, d_ff=2048, vocab=64, max_len=64)
    init = M.init_params(cfg, seed=0)
    x, dy = _tbase_layer_inputs()
    params16 = {k: v.half() for k, v in init.items()}
    w = M.EncoderLayerWeights.from_params(params16, "enc0.")
    lens = np.array([64, 60, 33, 64, 1, 64, 48, 64])
    mask = M.AttentionMask("padding", torch.tensor(lens, device="cuda"))
    y, stash = M.encoder_layer_forward(torch.tensor(x, device="cuda").half(), w, mask, 0.1, 99,
                                       n_heads=8)
    sink = M.GradSink()
    dx = M.encoder_layer_backward(torch.tensor(dy, device="cuda").half(), w, stash, sink,
                                  n_heads=8, p_drop=0.1, param_prefix="enc0.")
    P = {k: v.float().cpu().numpy() for k, v in params16.items()}
    ora = O.OracleTransformer(1, 1, 512, 8, 2048, 64, 64)
    yo, c = ora.enc_fwd(x.astype(np.float16).astype(np.float32), P, "enc0.",
                        O.pad_keep(lens, 64, 64), 0.1, 99, 0, np.float32)
    G = {}
    dxo = ora.enc_bwd(dy.astype(np.float16).astype(np.float32), c, P, "enc0.", 0.1, G, np.float32)
    assert np.abs(H(y).astype(np.float32) - yo).max() <= 2e-2 * np.abs(yo).max()
    assert np.abs(H(dx).astype(np.float32) - dxo).max() <= 2e-2 * np.abs(dxo).max()
    errs = {}
    for name, ref in G.items():
        got = H(sink.store[name]).astype(np.float64)
        errs[name] = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-12)
    # Normwise 2e-2 everywhere except the relu bias: its column sums inherit sign
    # flips of (x + b1) for pre-activations within fp16 rounding of 0 (the oracle
    # keeps u2 in f32), a few O(|dz|) terms per column -> a few percent.
    for name, e in errs.items():
        assert e <= (6e-2 if name.endswith("ffn.b1") else 2e-2), (name, e, errs)


def test_packed_kv_and_ordering():
    cfg = M.ModelConfig(n_enc=1, n_dec=2, d_model=8, n_heads=2, d_ff=16, vocab=11, max_len=6)
    tf = M.Transformer(cfg)
    params = tf.init_params(seed=1)
    rng = np.random.default_rng(5)
    batch = M.Batch(rng.integers(2, 11, (2, 5)), rng.integers(2, 11, (2, 5)),
                    rng.integers(2, 11, (2, 5)), np.array([5, 4]), 0)
    trace = []
    tf.forward_backward(params, batch, sink=M.GradSink(), trace=trace)
    assert trace.index(("enc_out_grad_emitted",)) > trace.index(("dec_layer_backward_done", 0))
    pw = M.pack_cross_weights([np.array([[2.0]])], [np.array([[4.0]])], [np.zeros(1)], [np.zeros(1)])
    x = np.full((1, 3, 1), 1.0)
    dx, dw, db = M.packed_kv_backward([np.ones((1, 3, 1))], [np.ones((1, 3, 1))], x, pw)
    assert np.allclose(H(dx), 6.0) and np.allclose(H(dw).ravel(), [3.0, 3.0])
    assert np.allclose(H(db).ravel(), [3.0, 3.0])
    with pytest.raises(IncompleteGradientSet):
        M.packed_kv_backward([np.zeros((1, 1, 1)), None], [np.zeros((1, 1, 1))] * 2,
                             np.zeros((1, 1, 1)), M.pack_cross_weights([np.eye(1)] * 2, [np.eye(1)] * 2,
                                                                       [np.zeros(1)] * 2, [np.zeros(1)] * 2))


def test_padding_positions_do_not_affect_loss_or_grads():
    cfg = M.ModelConfig(n_enc=1, n_dec=1, d_model=8, n_heads=2, d_ff=16, vocab=11, max_len=6)
    tf = M.Transformer(cfg)
    params = {k: v.double() for k, v in tf.init_params(seed=4).items()}
    rng = np.random.default_rng(11)
    src = rng.integers(2, 11, (2, 5))
    batch = M.Batch(src, rng.integers(2, 11, (2, 5)), rng.integers(2, 11, (2, 5)),
                    np.array([3, 2]), 0)
    s1 = M.GradSink()
    o1 = tf.forward_backward(params, batch, alpha=0.1, sink=s1)
    src2 = src.copy()
    src2[0, 3:] = 7
    src2[1, 2:] = 7
    s2 = M.GradSink()
    o2 = tf.forward_backward(params, M.Batch(src2, batch.tgt_in, batch.tgt_out, batch.src_len, 0),
                             alpha=0.1, sink=s2)
    assert o1.loss_sum == o2.loss_sum
    for name in s1.store:
        if name != "tok_emb":
            assert torch.equal(s1.store[name], s2.store[name]), name


def _tiny_run(graphs: bool, steps: int, p_drop=0.1):
    run = RunConfig()
    run.train.p_drop = p_drop
    run.train.cuda_graphs = graphs
    run.train.steps = steps
    eng = TrainingEngine(run)
    eng.setup_arena()
    ms = [eng.train_step(s) for s in range(steps)]
    return eng, ms


def test_engine_graph_replay_matches_eager():
    e1, m1 = _tiny_run(False, 12)
    e2, m2 = _tiny_run(True, 12)
    assert e2._graphs, "graphs were captured"
    for a, b in zip(m1, m2):
        assert abs(a.loss - b.loss) <= 1e-3 * max(1.0, abs(a.loss)), (a.step, a.loss, b.loss)
    p1, p2 = H(e1.ws.params16).astype(np.float32), H(e2.ws.params16).astype(np.float32)
    assert np.abs(p1 - p2).max() <= 2e-2
    assert e2.arena.realloc_count == 0 and e2.arena.high_water <= e2.capacity


def test_engine_trajectory_tracks_reference():
    """400 steps of the default copy-task job (p_drop 0.1) vs the reference
    engine's own trajectory (tests/golden/traj.npz): same batches, same dropout
    masks; fp16 workspace both sides, fp16 activations here."""
    import os
    from conftest import GOLDEN
    ref = np.load(os.path.join(GOLDEN, "traj.npz"))
    run = RunConfig()
    run.train.p_drop = 0.1
    eng = TrainingEngine(run)
    eng.setup_arena()
    losses = np.array([eng.train_step(s).loss for s in range(400)])
    want = ref["losses"]
    assert abs(losses[0] - want[0]) <= 2e-3 * want[0]
    for a in range(0, 400, 50):
        got_w, want_w = losses[a:a + 50].mean(), want[a:a + 50].mean()
        assert abs(got_w - want_w) <= 3e-2 * want_w, (a, got_w, want_w)
    assert abs(eng.evaluate() - float(ref["eval_acc"][0])) <= 0.06


def test_checkpoint_resume_bit_exact(tmp_path):
    run = RunConfig()
    run.train.p_drop = 0.1
    a = TrainingEngine(run)
    a.setup_arena()
    for s in range(6):
        a.train_step(s)
    a.save(str(tmp_path / "c.bin"), 6)
    for s in range(6, 10):
        a.train_step(s)
    b = TrainingEngine(run)
    b.setup_arena()
    assert b.restore(str(tmp_path / "c.bin")) == 6
    for s in range(6, 10):
        b.train_step(s)
    pa, pb = H(a.ws.params16).astype(np.float32), H(b.ws.params16).astype(np.float32)
    assert np.abs(pa - pb).max() <= 2e-3     # atomics only


def test_resume_from_a_reference_written_checkpoint(tmp_path):
    """Interop with F/checkpoint.py + F/engine.py:189-208: the reference engine's own
    LSF2 checkpoint of the default job after 40 steps (tests/golden/make_golden_ckpt.py)
    restores into this engine, which then continues the reference's uninterrupted
    trajectory (same batches, same dropout masks; fp16 activations here, fp32 there);
    and this engine's checkpoint carries the reference's tensor names, dtypes and
    shapes, so the reference can resume from it (T/test_data_cli.py:262-282)."""
    import os
    from conftest import GOLDEN
    from paper_2110_05722_b200.checkpoint import load_checkpoint
    ref = np.load(os.path.join(GOLDEN, "ref_ckpt_tail.npz"))
    path = os.path.join(GOLDEN, "ref_ckpt_step40.lsf2")
    run = RunConfig()
    run.train.p_drop = 0.1
    eng = TrainingEngine(run)
    eng.setup_arena()
    assert eng.restore(path) == 40 and eng.applied_steps == 40
    _, want_t = load_checkpoint(path)
    assert np.array_equal(H(eng.ws.params16).view(np.uint16), want_t["params16"].view(np.uint16))
    losses = np.array([eng.train_step(s).loss for s in range(40, 48)])
    assert np.abs(losses - ref["losses"]).max() <= 5e-3 * ref["losses"].max(), (losses, ref["losses"])
    assert eng.applied_steps == int(ref["applied"][0])
    p, q = H(eng.ws.params16).astype(np.float32), ref["params16"].astype(np.float32)
    assert np.linalg.norm(p - q) <= 1e-2 * np.linalg.norm(q)
    eng.save(str(tmp_path / "ours.lsf2"), 48)
    step, ours = load_checkpoint(str(tmp_path / "ours.lsf2"))
    assert step == 48 and list(ours) == list(want_t)
    for k in want_t:
        assert ours[k].dtype == want_t[k].dtype and ours[k].shape == want_t[k].shape, k
    assert float(ours["applied_steps"][0]) == 48.0


def test_tbase_step_runs_and_is_finite():
    from paper_2110_05722_b200.config import transformer_base
    from paper_2110_05722_b200.data import FixedShapeTask
    run = RunConfig(model=transformer_base(), train=TrainConfig(p_drop=0.1, batch_tokens=4096))
    eng = TrainingEngine(run, task=FixedShapeTask(64, 64, 32000))
    eng.setup_arena()
    ms = [eng.train_step(s) for s in range(4)]
    assert all(np.isfinite(m.loss) for m in ms) and ms[0].tokens == 4096
    assert abs(ms[0].loss - math.log(32000)) < 1.0
    assert not ms[-1].skipped


def _dp_run(force: bool, graphs: bool, steps: int, bucket_bytes=8 << 20, model=None, task=None,
            mode="shard", merge=True):
    from paper_2110_05722_b200.dist import DataParallel
    run = RunConfig() if model is None else RunConfig(model=model,
                                                      train=TrainConfig(p_drop=0.1,
                                                                        batch_tokens=4096))
    run.train.p_drop = 0.1
    run.train.cuda_graphs = graphs
    dp = DataParallel(bucket_bytes=bucket_bytes, force=force, mode=mode)
    eng = TrainingEngine(run, task=task, dp=dp)
    eng.merge_spans = merge
    eng.setup_arena()
    ms = [eng.train_step(s) for s in range(steps)]
    return eng, ms


@pytest.mark.parametrize("bucket_bytes,mode,merge", [(1 << 10, "shard", True), (8 << 20, "shard", True),
                                                     (1 << 10, "shard", False),
                                                     (8 << 20, "shard", False),
                                                     (1 << 10, "allreduce", True),
                                                     (8 << 20, "allreduce", True)])
def test_dp_exchange_one_rank_matches_local_step(bucket_bytes, mode, merge):
    """The overlapped exchange (per-bucket fp32 finish + NCCL reduce-scatter or
    all-reduce + narrow + non-finite count on the comm stream, then the sharded
    Adam and the params16 all-gather; one-rank communicator) inside the captured
    graph gives the local step's result: losses equal, parameters equal up to
    the embedding-scatter atomics."""
    e1, m1 = _dp_run(False, True, 8)
    e2, m2 = _dp_run(True, True, 8, bucket_bytes, mode=mode, merge=merge)
    assert e2._graphs and e2.dp.comm is not None
    for a, b in zip(m1, m2):
        assert a.tokens == b.tokens and a.skipped == b.skipped
        assert abs(a.loss - b.loss) <= 1e-4 * max(1.0, abs(a.loss)), (a.step, a.loss, b.loss)
    p1, p2 = H(e1.ws.params16).astype(np.float32), H(e2.ws.params16).astype(np.float32)
    assert np.abs(p1 - p2).max() <= 2e-3
    assert np.mean(p1 != p2) < 1e-2


def test_dp_exchange_buckets_cover_workspace_in_reverse_order():
    e, _ = _dp_run(True, False, 1, 1 << 10)
    plan = e._xplan
    assert plan.frontier == 0 and plan.issued == 0
    # finish order == reverse layout order: the planner never saw a gap
    offs = [lk.offset for lk in e.ws.links]
    assert offs == sorted(offs)


def test_dp_exchange_tbase_graph_step():
    """T-base shapes through the overlapped exchange + graph capture."""
    from paper_2110_05722_b200.config import transformer_base
    from paper_2110_05722_b200.data import FixedShapeTask
    e1, m1 = _dp_run(False, True, 4, model=transformer_base(), task=FixedShapeTask(64, 64, 32000))
    e2, m2 = _dp_run(True, True, 4, model=transformer_base(), task=FixedShapeTask(64, 64, 32000))
    assert e2.dp.sharded and e2._shard_spans
    for a, b in zip(m1, m2):
        assert abs(a.loss - b.loss) <= 1e-3 * abs(a.loss)
    p1, p2 = H(e1.ws.params16).astype(np.float32), H(e2.ws.params16).astype(np.float32)
    assert np.abs(p1 - p2).max() <= 2e-3


def _run_steps(steps, graphs=True):
    run = RunConfig()
    run.train.p_drop = 0.1
    run.train.cuda_graphs = graphs
    eng = TrainingEngine(run)
    eng.setup_arena()
    return eng, [eng.train_step(s) for s in steps]


@pytest.mark.parametrize("graphs,early", [(True, "1"), (False, "1"), (True, "0"), (True, "opt"),
                                          (False, "opt")])
def test_mask_bank_step_equals_inline_masks(monkeypatch, graphs, early):
    """Engine with the mask bank (every site drawn by one launch, step t+1's bits
    drawn beside step t's Adam) vs inline drawing: same masks, so the same
    losses; parameters equal up to embedding atomics.  The step sequence has
    gaps, so both the early draw and the in-step fallback are exercised."""
    steps = [0, 1, 2, 5, 6, 7, 9]
    monkeypatch.setenv("LS2_MASK_BANK", "0")
    e1, m1 = _run_steps(steps, graphs)
    monkeypatch.setenv("LS2_MASK_BANK", "1")
    monkeypatch.setenv("LS2_EARLY_MASKS", early)
    e2, m2 = _run_steps(steps, graphs)
    assert e1.masks is None and e2.masks is not None and e2.masks.buf is not None
    for a, b in zip(m1, m2):
        assert abs(a.loss - b.loss) <= 1e-4 * max(1.0, abs(a.loss)), (a.step, a.loss, b.loss)
    p1, p2 = H(e1.ws.params16).astype(np.float32), H(e2.ws.params16).astype(np.float32)
    assert np.abs(p1 - p2).max() <= 2e-3


def test_engine_wmt_shaped_buckets():
    """Variable-shape batches (WMT-shaped synthetic task): one
    planned arena for every bucket, one graph per bucket, no reallocation."""
    from paper_2110_05722_b200.config import transformer_base
    from paper_2110_05722_b200.data import WmtShapedTask
    run = RunConfig(model=transformer_base(32000, 256),
                    train=TrainConfig(p_drop=0.1, batch_tokens=4096))
    task = WmtShapedTask(4096, 64, 32000, seed=5)
    eng = TrainingEngine(run, task=task)
    eng.setup_arena()
    ms = [eng.train_step(s) for s in range(24)]
    assert all(np.isfinite(m.loss) for m in ms)
    assert len(eng._graphs) >= 3
    assert eng.arena.realloc_count == 0 and eng.arena.high_water <= eng.capacity
    # a replayed bucket gives the same loss as an eager run of the same batch
    assert all(m.tokens == int((np.asarray(task.batch(m.step).tgt_out) != 0).sum()) for m in ms)


def test_engine_file_task(tmp_path):
    """Token-file task (F/data.py:105-155) through the engine: bucketed batches,
    copy objective, loss falls."""
    rng = np.random.default_rng(0)
    lines = [" ".join(str(int(t)) for t in rng.integers(2, 19, rng.integers(3, 8)))
             for _ in range(64)]
    path = tmp_path / "tok.txt"
    path.write_text("\n".join(lines) + "\n")
    run = RunConfig()
    run.data.task, run.data.path = "file", str(path)
    run.train.p_drop = 0.0
    eng = TrainingEngine(run)
    eng.setup_arena()
    ms = [eng.train_step(s) for s in range(60)]
    assert all(np.isfinite(m.loss) for m in ms)
    assert np.mean([m.loss for m in ms[-8:]]) < np.mean([m.loss for m in ms[:8]])


@pytest.mark.parametrize("group", ["0", "3"])
def test_wgrad_batch_matches_per_layer_gemms(monkeypatch, group):
    """Weight gradients batched across layers (model._WgradBatch: pointer-array
    cuBLAS batches, flushed at the end of backward or every 3 layers, the
    readiness of their layers postponed) vs one GEMM per weight (LS2_WGRAD_BATCH=0):
    the same products, so losses agree and parameters agree up to fp32 summation
    order and the embedding atomics; T-base shapes, captured graphs."""
    from paper_2110_05722_b200.config import transformer_base
    from paper_2110_05722_b200.data import FixedShapeTask

    def run(env):
        monkeypatch.setenv("LS2_WGRAD_BATCH", env)
        cfg = RunConfig(model=transformer_base(), train=TrainConfig(p_drop=0.1, batch_tokens=4096))
        eng = TrainingEngine(cfg, task=FixedShapeTask(64, 64, 32000))
        eng.setup_arena()
        return eng, [eng.train_step(s) for s in range(4)]

    e1, m1 = run("0")
    e2, m2 = run("auto" if group == "0" else group)
    assert e1.wgrad_group is None and e2.wgrad_group == int(group)
    for a, b in zip(m1, m2):
        assert abs(a.loss - b.loss) <= 1e-4 * abs(a.loss), (a.step, a.loss, b.loss)
        assert not b.skipped
    g1, g2 = H(e1.ws.grads16).astype(np.float32), H(e2.ws.grads16).astype(np.float32)
    assert np.linalg.norm(g1 - g2) <= 1e-3 * np.linalg.norm(g1)
    p1, p2 = H(e1.ws.params16).astype(np.float32), H(e2.ws.params16).astype(np.float32)
    assert np.abs(p1 - p2).max() <= 2e-3
    assert e2.arena.realloc_count == 0 and e2.arena.high_water <= e2.capacity
