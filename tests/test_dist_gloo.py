"""Data-parallel semantics on CPU with gloo (world sizes 2 and 4, 127.0.0.1).

Each rank runs the oracle step on its share of the batch and then the exact DP
recipe of paper_2110_05722_b200.dist / engine._exchange_bucket / _dp_update:
  totals all-reduce -> reverse-order fp32 buckets (aligned starts) ->
  reduce-scatter ("shard") or all-reduce ("allreduce") in fp32 -> narrow the
  reduced chunk by loss_scale / GLOBAL token count -> global non-finite count
  -> Adam on the rank's chunks -> all-gather params16 ("shard").
The N-rank result must equal the 1-rank step on the concatenated batch within
fp16 tolerance (in fact almost bit for bit: only the fp32 summation order
differs), and every rank must hold bit-identical parameters.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lsport as O

CFG = dict(n_enc=1, n_dec=1, d=16, heads=4, dff=24, vocab=19, max_len=8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup():
    shapes = O.model_param_shapes(CFG["n_enc"], CFG["n_dec"], CFG["d"], CFG["dff"], CFG["vocab"],
                                  CFG["max_len"])
    init = O.model_init(shapes, 3)
    p16 = np.concatenate([O.to_half(init[n].reshape(-1)) for n, _ in shapes])
    rng = np.random.default_rng(9)
    b, l = 4, 6
    batch = (rng.integers(2, 19, (b, l)), rng.integers(2, 19, (b, l)), rng.integers(2, 19, (b, l)),
             np.array([6, 5, 3, 6]))
    batch[2][1, 4:] = 0      # some pad targets: per-rank token counts differ
    model = O.OracleTransformer(CFG["n_enc"], CFG["n_dec"], CFG["d"], CFG["heads"], CFG["dff"],
                                CFG["vocab"], CFG["max_len"])
    return shapes, p16, batch, model


def _grads(model, shapes, p16, batch):
    P, off = {}, 0
    for name, shp in shapes:
        n = int(np.prod(shp))
        P[name] = p16[off:off + n].reshape(shp)
        off += n
    src, tin, tout, lens = batch
    loss, cnt, _, G = model.forward_backward(P, src, tin, tout, lens, pad_id=0, p=0.0, alpha=0.1)
    return loss, cnt, np.concatenate([np.asarray(G[n], np.float32).reshape(-1) for n, _ in shapes])


def _worker(rank, world, port, mode, poison, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_05722_b200.dist import DataParallel
    dp = DataParallel(bucket_bytes=512, mode=mode)        # many buckets
    shapes, p16, batch, model = _setup()
    per = 4 // world
    part = [x[rank * per:(rank + 1) * per] for x in batch]
    loss, cnt, acc = _grads(model, shapes, p16, part)
    if poison and rank == world - 1:
        acc[7] = np.inf                     # one rank's gradient overflows
    totals = torch.tensor([loss, float(cnt), 0.0], dtype=torch.float64)
    dp.allreduce_totals(totals)
    scale = np.float32(4.0 / totals[1].item())          # loss_scale 4 / global count
    n = p16.size
    n_pad = dp.padded(n)
    acc32 = torch.zeros(n_pad, dtype=torch.float32)
    acc32[:n] = torch.from_numpy(acc)
    links, off = [], 0
    for name, shp in shapes:
        links.append((name, off, int(np.prod(shp))))
        off += int(np.prod(shp))
    plan = dp.exchange_plan(links, n)
    spans = []
    for name, _, _ in reversed(links):          # backward finishes in reverse order
        spans += plan.ready([name])
    spans += plan.flush()
    g16 = np.zeros(n_pad, np.float16)
    chunks = []
    bad = 0
    for s, e in spans:
        if dp.sharded:
            dp.reduce_scatter_span(acc32, s, e)
        else:
            dp.allreduce_span(acc32, s, e)
        o, c = dp.chunk(s, e)
        g16[o:o + c] = O.to_half(acc32[o:o + c].numpy() * scale)
        bad += int(np.count_nonzero(~np.isfinite(O.from_half(g16[o:o + c]))))
        chunks.append((o, c))
    nf = torch.tensor([bad], dtype=torch.int32)
    if dp.sharded:
        dp.allreduce_count(nf)
    pp = np.zeros(n_pad, np.float16)
    pp[:n] = p16
    m = np.zeros(n_pad, np.float32)
    v = np.zeros(n_pad, np.float32)
    if int(nf.item()) == 0:
        for o, c in chunks:
            assert O.adam_flat(pp[o:o + c], g16[o:o + c], m[o:o + c], v[o:o + c], lr=1e-2,
                               beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0, loss_scale=4.0,
                               t=1) == 0
    if dp.sharded:
        pt = torch.from_numpy(pp)
        for s, e in spans:
            dp.all_gather_span(pt, s, e)
        pp = pt.numpy()
    out_q.put((rank, totals.numpy().tolist(), pp[:n].copy(), int(nf.item()), spans, n_pad))
    dist.barrier()
    dist.destroy_process_group()


def _run_ranks(world, mode, poison=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, poison, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,mode", [(2, "shard"), (4, "shard"), (2, "allreduce"),
                                        (4, "allreduce")])
def test_n_rank_step_equals_one_rank_step(world, mode):
    res = _run_ranks(world, mode)
    _, tot0, p0, bad0, buckets, n_pad = res[0]
    for _, tot, p, bad, _, _ in res[1:]:
        assert bad == bad0 == 0
        assert np.array_equal(p.view(np.uint16), p0.view(np.uint16))   # identical replicas
        assert tot == tot0
    # buckets: contiguous reverse-order cover of the padded workspace, aligned starts
    align = 64 * (world if mode == "shard" else 1)
    assert n_pad % align == 0 and n_pad >= p0.size
    spans = sorted(buckets)
    assert spans[0][0] == 0 and spans[-1][1] == n_pad and buckets[0][1] == n_pad
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert all(s % align == 0 and (e - s) % align == 0 for s, e in buckets)
    # single-rank reference on the concatenated batch
    shapes, p16, batch, model = _setup()
    loss, cnt, acc = _grads(model, shapes, p16, batch)
    assert cnt == int(tot0[1]) and abs(loss - tot0[0]) <= 1e-5 * abs(loss)
    g16 = O.to_half(acc * np.float32(4.0 / cnt))
    m = np.zeros(p16.size, np.float32)
    v = np.zeros(p16.size, np.float32)
    O.adam_flat(p16, g16, m, v, lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0,
                loss_scale=4.0, t=1)
    diff = np.abs(p0.astype(np.float32) - p16.astype(np.float32))
    assert diff.max() <= 2e-2 * max(1.0, np.abs(p16.astype(np.float32)).max())
    # the fp32 sum differs from the one-rank gradient only in summation order:
    # nearly every updated parameter is bit-identical
    assert np.mean(p0 != p16) < 0.02


@pytest.mark.parametrize("mode", ["shard", "allreduce"])
def test_non_finite_gradient_on_one_rank_skips_everywhere(mode):
    res = _run_ranks(2, mode, poison=True)
    shapes, p16, _, _ = _setup()
    for _, _, p, bad, _, _ in res:
        assert bad > 0
        assert np.array_equal(p.view(np.uint16), p16.view(np.uint16))    # no update anywhere


def test_rank_sharded_task_interleaves_the_stream():
    from paper_2110_05722_b200.config import RunConfig
    from paper_2110_05722_b200.data import make_task
    from paper_2110_05722_b200.dist import RankShardedTask
    cfg = RunConfig()
    base = make_task(cfg)
    shards = [RankShardedTask(base, r, 3) for r in range(3)]
    for step in range(3):
        for r, t in enumerate(shards):
            a, b = t.batch(step), base.batch(step * 3 + r)
            assert np.array_equal(a.src, b.src) and np.array_equal(a.tgt_out, b.tgt_out)
    assert shards[0].possible_shapes() == base.possible_shapes()


def test_grad_exchange_plan_reverse_suffix_buckets():
    from paper_2110_05722_b200.dist import GradExchange
    links = [("a", 0, 10), ("b", 10, 5), ("c", 15, 20), ("d", 35, 5)]
    x = GradExchange(links, 40, bucket_elems=8)
    assert x.ready(["d"]) == []                 # 5 pending < 8
    assert x.ready(["b"]) == []                 # not a suffix yet (c missing)
    assert x.ready(["c"]) == [(10, 40)]          # c and b join the suffix
    with pytest.raises(RuntimeError):
        GradExchange(links, 40, 8).flush()       # nothing finished
    x.reset()
    out = x.ready(["d", "c", "b", "a"])
    assert out == [(0, 40)] and x.flush() == []


def test_grad_exchange_plan_small_buckets_cover_exactly():
    from paper_2110_05722_b200.dist import GradExchange
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 50, 30)
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    links = [(f"p{i}", int(o), int(s)) for i, (o, s) in enumerate(zip(offs, sizes))]
    n = int(sizes.sum())
    x = GradExchange(links, n, bucket_elems=40)
    spans = []
    for i in reversed(range(30)):
        spans += x.ready([f"p{i}"])
    spans += x.flush()
    assert spans[0][1] == n and spans[-1][0] == 0
    assert all(a[0] == b[1] for a, b in zip(spans, spans[1:]))
    assert all(e - s >= 40 for s, e in spans[:-1])


def _warm_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2110_05722_b200.data import WmtShapedTask
    from paper_2110_05722_b200.dist import DataParallel

    class FakeEngine:
        """train_step = the first step of a new bucket records its graph; every step
        runs one all-reduce (the gradient exchange) like the real DP step."""
        device = None

        def __init__(self, task):
            self.task, self._graphs, self.steps = task, {}, 0

        def train_step(self, s):
            key = ("train",) + tuple(np.asarray(self.task.batch(s).src).shape)
            self._graphs.setdefault(key, True)
            t = torch.ones(1)
            dist.all_reduce(t)
            assert t.item() == world
            self.steps += 1

    task = WmtShapedTask(4096, 64, 32000, seed=17 + rank)   # per-rank bucket sequences
    eng = FakeEngine(task)
    keys = [("train",) + tuple(sh) for sh in task.possible_shapes()]
    n = bench.warm_up(eng, keys, 3, DataParallel())
    out_q.put((rank, n, eng.steps, all(k in eng._graphs for k in keys)))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_warm_up_stops_together_on_all_ranks():
    """WMT-shaped data draws a different bucket sequence per rank; the bench's
    warm-up must stop on the same step everywhere (a max over ranks), or the rank
    that finished first leaves the others blocked in the gradient all-reduce."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_warm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, n0, s0, all0), (_, n1, s1, all1) = res
    assert n0 == n1 == s0 == s1 and all0 and all1
