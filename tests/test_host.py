"""CPU-only tests: the C-ABI library loads and exports every symbol declared in
include/ls2.h, host-side planner/arena logic (F/memplan.py semantics, pinned by
golden plans), configs, data and the LSF2 checkpoint format."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "ls2.h")).read()
    return sorted(set(re.findall(r"\b(ls2_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    import torch  # noqa: F401
    from paper_2110_05722_b200 import _lib
    lib = _lib.load_library()
    syms = _header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.exported_symbols())
    assert lib.ls2_version() == 1


def test_library_host_queries_without_gpu():
    import torch  # noqa: F401
    from paper_2110_05722_b200 import _lib
    _lib.load_library()
    assert _lib.call_i64("ls2_colsum_ws_bytes", 4096, 512) == 148 * 512 * 8
    assert _lib.call_i64("ls2_layernorm_bwd_ws_bytes", 4096, 512) == 148 * 3 * 512 * 8
    assert _lib.call_i64("ls2_gemm_scratch_bytes", 64, 8) == 3 * 512 * 8


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch
    from paper_2110_05722_b200 import _lib
    from paper_2110_05722_b200.errors import DeviceError
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(DeviceError):
        _lib.context()


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2110_05722_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f


# --- planner -------------------------------------------------------------------------

def test_plan_matches_reference_golden(golden_ops):
    from paper_2110_05722_b200.memplan import Lifetime, plan, simulate_plan_safety
    lts = [Lifetime(*(int(v) for v in r)) for r in golden_ops["plan_in"]]
    p = plan(lts)
    assert p.blocks == list(golden_ops["plan_blocks"])
    assert [p.assignment[i] for i in range(40)] == list(golden_ops["plan_assign"])
    assert simulate_plan_safety(p).ok


def test_attention_backward_paper_bound():
    from paper_2110_05722_b200.memplan import (PlanShape, attention_backward_lifetimes,
                                               naive_attention_backward_peak, plan)
    for b, h, l, n in [(1, 4, 2, 1), (8, 256, 32, 4), (3, 7, 9, 2), (2, 4, 32, 8)]:
        sh = PlanShape(b, h, l, n)
        p = plan(attention_backward_lifetimes(sh))
        assert p.peak == 3 * b * h * l + max(3 * b * h * l, b * l * l * n)
        assert p.peak <= naive_attention_backward_peak(sh)
    assert plan(attention_backward_lifetimes(PlanShape(1, 4, 2, 1))).peak == 48


def test_plan_fuzz_safe_and_permutation_invariant():
    from paper_2110_05722_b200.memplan import Lifetime, naive_peak, plan, simulate_plan_safety
    rng = np.random.default_rng(6)
    for _ in range(300):
        n = int(rng.integers(1, 24))
        lts = []
        for i in range(n):
            f = int(rng.integers(0, 40))
            lts.append(Lifetime(i, int(rng.integers(1, 100)), f, f + int(rng.integers(0, 15))))
        p = plan(lts)
        assert simulate_plan_safety(p).ok and p.peak <= naive_peak(lts)
        q = plan([lts[i] for i in rng.permutation(n)])
        assert q.blocks == p.blocks and q.assignment == p.assignment


def test_simulator_flags_overlap_and_classify():
    from paper_2110_05722_b200.errors import ShapeMismatch, UntaggedTensor
    from paper_2110_05722_b200.memplan import (Lifetime, MemoryPlan, TensorTag, classify,
                                               simulate_plan_safety)
    lts = [Lifetime(0, 4, 0, 3), Lifetime(1, 4, 2, 5)]
    assert not simulate_plan_safety(MemoryPlan([4], {0: 0, 1: 0}, lts)).ok
    assert classify([TensorTag("w", "parameter"), TensorTag("x", "activation")]) == \
        {"w": "permanent", "x": "temporary"}
    with pytest.raises(UntaggedTensor):
        classify([TensorTag("x", "mystery")])
    with pytest.raises(ShapeMismatch):
        Lifetime(0, 0, 0, 1)


# --- config / data / checkpoint -------------------------------------------------------

def test_config_validation_and_json(tmp_path):
    import json
    from paper_2110_05722_b200.config import RunConfig, load_run_config
    from paper_2110_05722_b200.errors import ConfigError
    from paper_2110_05722_b200.model import ModelConfig
    from paper_2110_05722_b200.trainer import OptimConfig
    with pytest.raises(ConfigError):
        ModelConfig(d_model=10, n_heads=4)
    with pytest.raises(ConfigError):
        OptimConfig(loss_scale=3.0)
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"model": {"d_model": 64, "n_heads": 4}, "train": {"lr": 1e-3}}))
    rc = load_run_config(str(p))
    assert rc.model.d_model == 64 and rc.train.lr == 1e-3
    p.write_text(json.dumps({"model": {"bogus": 1}}))
    with pytest.raises(ConfigError):
        load_run_config(str(p))
    assert RunConfig().echo()["model"]["n_heads"] == 4


def test_synthetic_task_pure_function_of_seed_step():
    from paper_2110_05722_b200.config import RunConfig
    from paper_2110_05722_b200.data import FixedShapeTask, SyntheticTask
    t = SyntheticTask(RunConfig())
    a, b = t.batch(5), t.batch(5)
    assert np.array_equal(a.src, b.src) and np.array_equal(a.tgt_in, b.tgt_in)
    assert a.src.shape[1] % 4 == 0 and (a.src.shape[0], a.src.shape[1]) in t.possible_shapes()
    assert np.array_equal(a.tgt_out[a.src != 0], a.src[a.src != 0])
    f = FixedShapeTask(64, 64, 32000).batch(3)
    assert f.src.shape == (64, 64) and f.src.min() >= 2 and f.src.max() < 32000
    assert np.array_equal(f.tgt_in[:, 1:], f.tgt_out[:, :-1])


def test_synthetic_task_matches_reference_semantics():
    """Same draws as F/data.py:83-102 (counter RNG), checked against the oracle RNG."""
    from oracle import lsport as O
    from paper_2110_05722_b200.data import _uniform
    assert np.array_equal(_uniform(12345, 100), O.counter_uniform(12345, 0, 100))


def test_checkpoint_roundtrip(tmp_path):
    from paper_2110_05722_b200.checkpoint import load_checkpoint, save_checkpoint
    from paper_2110_05722_b200.errors import ParseError
    p16 = np.random.default_rng(0).normal(size=(7,)).astype(np.float16)
    m = np.arange(7, dtype=np.float32)
    save_checkpoint(str(tmp_path / "a.bin"), 42, [("params16", p16), ("m", m)])
    step, t = load_checkpoint(str(tmp_path / "a.bin"))
    assert step == 42 and np.array_equal(t["params16"].view(np.uint16), p16.view(np.uint16))
    assert np.array_equal(t["m"], m)
    (tmp_path / "b.bin").write_bytes(b"XXXX")
    with pytest.raises(ParseError):
        load_checkpoint(str(tmp_path / "b.bin"))


def test_checkpoint_bytes_identical_to_the_reference_writer(tmp_path):
    """tests/golden/ref_ckpt_format.lsf2 was written by the reference's
    save_checkpoint (F/checkpoint.py:27-42) from fixed tensors (f16/f32, ranks 0-3,
    an empty tensor): this writer produces the same bytes and this reader
    recovers the same tensors; the reference engine's own checkpoint parses too."""
    import importlib.util
    from conftest import GOLDEN
    from paper_2110_05722_b200.checkpoint import load_checkpoint, save_checkpoint
    spec = importlib.util.spec_from_file_location(
        "make_golden_ckpt", os.path.join(GOLDEN, "make_golden_ckpt.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    tensors = gen.format_tensors()
    ref_path = os.path.join(GOLDEN, "ref_ckpt_format.lsf2")
    save_checkpoint(str(tmp_path / "ours.lsf2"), 123456789, tensors)
    assert (tmp_path / "ours.lsf2").read_bytes() == open(ref_path, "rb").read()
    step, got = load_checkpoint(ref_path)
    assert step == 123456789 and list(got) == [n for n, _ in tensors]
    for name, arr in tensors:
        assert got[name].dtype == arr.dtype and got[name].shape == arr.shape
        assert got[name].tobytes() == arr.tobytes()
    step, eng = load_checkpoint(os.path.join(GOLDEN, "ref_ckpt_step40.lsf2"))
    assert step == 40 and list(eng) == ["params16", "moments_m", "moments_v", "applied_steps"]
    assert eng["params16"].dtype == np.float16 and eng["moments_v"].dtype == np.float32
    assert eng["params16"].size == eng["moments_m"].size == eng["moments_v"].size


def test_oracle_never_imports_product():
    src = open(os.path.join(ROOT, "oracle", "lsport.py")).read()
    mods = re.findall(r"^\s*(?:from|import)\s+([\w.]+)", src, re.M)
    assert not any(m.startswith("paper_2110_05722_b200") for m in mods), mods


def test_file_task_matches_reference_golden(tmp_path):
    """FileTask (F/data.py:105-155) vs the reference's own batches on the same token
    file (tests/golden/data.npz, written by tests/golden/make_golden_data.py)."""
    import os
    from conftest import GOLDEN
    from paper_2110_05722_b200.config import RunConfig
    from paper_2110_05722_b200.data import FileTask
    g = np.load(os.path.join(GOLDEN, "data.npz"))
    path = tmp_path / "tokens.txt"
    path.write_bytes(g["file_text"].tobytes())
    run = RunConfig()
    run.model.vocab, run.model.max_len = 50, 24
    run.train.batch_tokens = 96
    run.data.task, run.data.path = "file", str(path)
    ft = FileTask(run)
    assert len(ft.batches) == int(g["file_n"][0])
    for i, b in enumerate(ft.batches):
        for k in ("src", "tgt_in", "tgt_out", "src_len"):
            assert np.array_equal(np.asarray(getattr(b, k)), g[f"file_{i}_{k}"]), (i, k)
    assert ft.possible_shapes() == sorted({g[f"file_{i}_src"].shape
                                           for i in range(int(g["file_n"][0]))})


@pytest.mark.parametrize("task", ["copy", "reverse"])
def test_synthetic_task_matches_reference_golden(task):
    import os
    from conftest import GOLDEN
    from paper_2110_05722_b200.config import RunConfig
    from paper_2110_05722_b200.data import SyntheticTask
    g = np.load(os.path.join(GOLDEN, "data.npz"))
    run = RunConfig()
    run.data.task = task
    st = SyntheticTask(run)
    for step in (0, 1, 7):
        b = st.batch(step)
        for k in ("src", "tgt_in", "tgt_out", "src_len"):
            assert np.array_equal(np.asarray(getattr(b, k)), g[f"{task}_{step}_{k}"]), (step, k)


def test_wmt_shaped_task_buckets_and_budget():
    from paper_2110_05722_b200.data import WmtShapedTask
    t = WmtShapedTask(4096, 64, 32000, seed=3)
    shapes = set(t.possible_shapes())
    seen = set()
    for s in range(40):
        b = t.batch(s)
        src = np.asarray(b.src)
        assert tuple(src.shape) in shapes
        assert src.shape[1] % 4 == 0 and src.size <= 4096
        lens = np.asarray(b.src_len)
        assert lens.min() >= 1 and lens.max() <= src.shape[1]
        assert np.all(src[np.arange(src.shape[1])[None, :] >= lens[:, None]] == 0)
        seen.add(tuple(src.shape))
        b2 = t.batch(s)
        assert np.array_equal(np.asarray(b2.src), src)      # pure function of step
    assert len(seen) > 4


def test_roofline_table_kernel_names_and_bounds():
    """bench.py's per-kernel roofline rows: the LayerNorm backward is matched under
    both kernel names, and the flash attention passes are reported against the
    tensor peak with their HBM fraction kept (paper_2110_05722_b200/roofline.py)."""
    from paper_2110_05722_b200 import roofline as RL
    algo = RL.algo_table(4096, 512, 2048, 32000, 64, 64, 8, 60_655_616)
    times = {
        "void ls2::ln_bwd_reg<__half, __half, float, 2, true, true, true>(a)": [28, 200.0],
        "void ls2::ln_bwd_stage<__half, __half, float, 2, true, true, true, false>(a)": [28, 210.0],
        "ls2::atc::attn_flash_dkv_kernel(a)": [12, 960.0],
        "nvjet_hsh_128x128_64x8_2x2_2cta_v_bz_NNT": [49, 340.0],
    }
    rows = RL.kernel_table(times, algo, 6545.0, flops=RL.tensor_flops(16, 512, 12, 768),
                           peak_tflops=1419.7)
    by = {r["kernel"].split("<")[0]: r for r in rows}
    assert set(by) == {"ln_bwd_reg", "ln_bwd_stage", "atc::attn_flash_dkv_kernel"}  # no cuBLAS rows
    assert by["ln_bwd_reg"]["bound"] == "hbm" and by["ln_bwd_reg"]["bytes_per_launch"] == \
        5 * 4096 * 512 * 2 + 4096 * 512 // 8 + 8 * 4096
    fl = by["atc::attn_flash_dkv_kernel"]
    assert fl["bound"] == "tensor" and fl["flops_per_launch"] == 4 * 2 * 16 * 12 * 512 * 512 * 64
    assert abs(fl["frac"] - fl["achieved_tflops"] / 1419.7) < 1e-3 and fl["hbm_frac"] < fl["frac"]
    assert [r["us_per_step"] for r in rows] == sorted((r["us_per_step"] for r in rows), reverse=True)
