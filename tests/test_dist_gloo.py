"""Data-parallel semantics on CPU with gloo (world_size 2, 127.0.0.1).

Each rank runs the oracle step on its half of the batch and then the exact DP
recipe of paper_2110_05722_b200.dist / engine._update:
  totals all-reduce -> scale by loss_scale / GLOBAL token count -> fp16 narrow
  -> bucketed fp16 all-reduce (reverse order) -> global non-finite check -> Adam.
The 2-rank result must equal the 1-rank step on the concatenated batch within
fp16 tolerance, and both ranks must hold bit-identical parameters.
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


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_05722_b200.dist import DataParallel
    dp = DataParallel(bucket_bytes=512)        # many buckets
    shapes, p16, batch, model = _setup()
    half = [x[rank * 2:(rank + 1) * 2] for x in batch]
    loss, cnt, acc = _grads(model, shapes, p16, half)
    totals = torch.tensor([loss, float(cnt), 0.0], dtype=torch.float64)
    dp.allreduce_totals(totals)
    scale = np.float32(4.0 / totals[1].item())          # loss_scale 4 / global count
    g16 = torch.from_numpy(O.to_half(acc * scale))
    # the engine's overlapped recipe: backward finishes parameters in reverse
    # layout order; each finished suffix bucket is all-reduced as it appears
    links, off = [], 0
    for name, shp in shapes:
        links.append((name, off, int(np.prod(shp))))
        off += int(np.prod(shp))
    plan = dp.exchange_plan(links, off, elem_bytes=2)
    spans = []
    for name, _, _ in reversed(links):
        spans += plan.ready([name])
    spans += plan.flush()
    for s, e in spans:
        dp.allreduce_span(g16, s, e)
    m = np.zeros(p16.size, np.float32)
    v = np.zeros(p16.size, np.float32)
    bad = O.adam_flat(p16, g16.numpy(), m, v, lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0,
                      loss_scale=4.0, t=1)
    out_q.put((rank, totals.numpy().tolist(), p16.copy(), bad, spans))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_step_equals_one_rank_step():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, tot0, p0, bad0, buckets), (_, tot1, p1, bad1, _) = res
    assert bad0 == bad1 == 0
    assert np.array_equal(p0.view(np.uint16), p1.view(np.uint16))   # identical replicas
    assert tot0 == tot1
    # buckets: contiguous cover in reverse layout order
    spans = sorted(buckets)
    assert spans[0][0] == 0 and spans[-1][1] == p0.size and buckets[0][1] == p0.size
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
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
    assert np.mean(p0 != p16) < 0.2


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
