"""CPU tests of the host logic that batches weight gradients across layers
(model._WgradBatch with model._ViewSink): which products are held back and
grouped by shape, when the arena frees of their operands happen, how the
readiness of the layers they belong to (the data-parallel exchange trigger) is
postponed to the flush, and that a second producer of a pending gradient
flushes it first.  The cuBLAS calls are replaced by torch CPU matmuls here;
tests/test_gpu_model.py::test_wgrad_batch_matches_per_layer_gemms runs the real
path on the B200."""

import pytest
import torch

from paper_2110_05722_b200 import model as M


class _Arena:
    def __init__(self):
        self.freed = []

    def free(self, t):
        self.freed.append(t.data_ptr())


@pytest.fixture
def fake_gemms(monkeypatch):
    calls = []

    def gemm_list(a_list, b_list, outs, trans_a=False, trans_b=False, alpha=1.0, beta=0.0):
        calls.append(("list", len(a_list), tuple(a_list[0].shape), beta))
        for a, b, o in zip(a_list, b_list, outs):
            o.mul_(beta).add_(alpha * (a.t() @ b))

    def gemm(a, b, trans_a=False, out=None, beta=0.0, **kw):
        calls.append(("single", tuple(a.shape)))
        out.mul_(beta).add_(a.t() @ b)
        return out

    monkeypatch.setattr(M.K, "gemm_list", gemm_list)
    monkeypatch.setattr(M.K, "gemm", gemm)
    return calls


def _sink(group, names_shapes):
    store = {n: torch.full(s, 7.0) for n, s in names_shapes.items()}
    sink = M._ViewSink(store, wgrad_group=group)
    ready = []
    sink.on_ready = lambda names: ready.append(None if names is None else sorted(names))
    return sink, store, ready


def test_batches_by_shape_holds_frees_and_postpones_readiness(fake_gemms):
    g = torch.Generator().manual_seed(0)
    shapes = {"l1.wo": (8, 8), "l1.w1": (16, 8), "l0.wo": (8, 8), "l0.w1": (16, 8)}
    sink, store, ready = _sink(0, shapes)
    arena = _Arena()
    lane, arena_f, join = M._open_lane(sink, arena, torch.float32)
    assert isinstance(lane, M._WgradBatch) and sink.lane is lane
    ops = {}
    for layer in ("l1", "l0"):
        for nm, (r, c) in (("wo", (8, 8)), ("w1", (16, 8))):
            dy, x = torch.randn(32, r, generator=g), torch.randn(32, c, generator=g)
            ops[f"{layer}.{nm}"] = (dy, x)
            M._wgrad(sink, f"{layer}.{nm}", dy, x)
            arena_f.free(dy)                 # held: the product has not run yet
            arena_f.free(x)
        join()
        M._ready(sink, f"{layer}.")
    assert fake_gemms == [] and arena.freed == [] and ready == []
    assert all(torch.equal(store[n], torch.full(s, 7.0)) for n, s in shapes.items())
    M._close_lane(sink, lane)
    # one batched call per shape, in first-seen order, then the postponed readiness
    assert fake_gemms == [("list", 2, (32, 8), 0.0), ("list", 2, (32, 16), 0.0)]
    assert ready == [["l1.w1", "l1.wo"], ["l0.w1", "l0.wo"]]
    assert len(arena.freed) == 8 and sink.lane is None
    for n, (dy, x) in ops.items():
        assert torch.allclose(store[n], dy.t() @ x)
    M._ready(sink, None)                     # nothing pending: immediate
    assert ready[-1] is None


def test_group_flushes_every_k_layers(fake_gemms):
    sink, store, ready = _sink(2, {f"l{i}.wo": (4, 4) for i in range(4)})
    lane, arena_f, join = M._open_lane(sink, _Arena(), torch.float32)
    for i in reversed(range(4)):
        M._wgrad(sink, f"l{i}.wo", torch.randn(8, 4), torch.randn(8, 4))
        join()
        M._ready(sink, f"l{i}.")
    # flushed after layers 3,2 and after 1,0: two batches of two
    assert [c[:2] for c in fake_gemms] == [("list", 2), ("list", 2)]
    assert ready == [["l3.wo"], ["l2.wo"], ["l1.wo"], ["l0.wo"]]


def test_second_producer_settles_the_pending_product(fake_gemms):
    sink, store, ready = _sink(0, {"tok_emb": (4, 4)})
    lane, arena_f, join = M._open_lane(sink, _Arena(), torch.float32)
    dy, x = torch.randn(8, 4), torch.randn(8, 4)
    M._wgrad(sink, "tok_emb", dy, x)           # small output: batched, pending
    assert "tok_emb" in lane.pending
    v, beta = sink.target("tok_emb")           # another producer accumulates now
    assert fake_gemms == [("list", 1, (8, 4), 0.0)] and beta == 1
    v.add_(1.0)
    assert torch.allclose(store["tok_emb"], dy.t() @ x + 1.0)


def test_large_outputs_run_at_once(fake_gemms, monkeypatch):
    monkeypatch.setattr(M._WgradBatch, "MAX_OUT", 15)
    sink, store, _ = _sink(0, {"big": (4, 4), "small": (2, 2)})
    lane, arena_f, join = M._open_lane(sink, _Arena(), torch.float32)
    M._wgrad(sink, "big", torch.randn(8, 4), torch.randn(8, 4))
    M._wgrad(sink, "small", torch.randn(8, 2), torch.randn(8, 2))
    assert fake_gemms == [("single", (8, 4))] and lane.pending == {"small"}


def test_float64_and_off_take_no_lane():
    sink, _, _ = _sink(0, {"w": (2, 2)})
    assert M._open_lane(sink, _Arena(), torch.float64)[0] is None
    sink2 = M._ViewSink({}, wgrad_group=None)
    assert M._open_lane(sink2, _Arena(), torch.float16)[0] is None
