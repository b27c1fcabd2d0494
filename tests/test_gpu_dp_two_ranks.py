"""The engine's multi-rank data-parallel step on real kernels: two processes share
cuda:0 and exchange through torch.distributed (gloo on CUDA tensors) instead of
NCCL, which refuses two ranks on one device.  This runs everything the one-rank
NCCL tests cannot: rank-specific bucket chunks (rank 1's chunks sit in the
middle of every bucket), the sharded Adam over non-adjacent spans
(`ls2_adam_spans`), the params16 all-gather, the scalar non-finite all-reduce
and the rank-interleaved batches (dist.RankShardedTask).  Eager steps (gloo
cannot be captured in a CUDA graph).
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, mode, steps, out_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2110_05722_b200.config import RunConfig
    from paper_2110_05722_b200.dist import DataParallel, RankShardedTask
    from paper_2110_05722_b200.engine import TrainingEngine
    run = RunConfig()
    run.train.p_drop = 0.1
    run.train.cuda_graphs = False
    dp = DataParallel(bucket_bytes=4 << 10, mode=mode, native=False)
    eng = TrainingEngine(run, dp=dp)
    assert isinstance(eng.task, RankShardedTask)
    eng.setup_arena()
    p0 = eng.ws.params16.cpu().numpy().copy()
    ms = [eng.train_step(s) for s in range(steps)]
    torch.cuda.synchronize()
    own = [int((np.asarray(eng.task.batch(s).tgt_out) != 0).sum()) for s in range(steps)]
    out_q.put((rank, eng.ws.params16.cpu().numpy().copy(), p0, [m.loss for m in ms],
               [m.tokens for m in ms], own, [m.skipped for m in ms], len(eng._buckets),
               sorted(eng._shard_spans)))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, mode, steps=4):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.fixture(scope="module")
def runs():
    return {mode: _run(2, mode) for mode in ("shard", "allreduce")}


@pytest.mark.parametrize("mode", ["shard", "allreduce"])
def test_two_ranks_keep_identical_replicas(runs, mode):
    (_, pa, p0, la, ta, own_a, sk_a, nb, spans_a), (_, pb, _, lb, tb, own_b, _, _, spans_b) = \
        runs[mode]
    assert np.array_equal(pa.view(np.uint16), pb.view(np.uint16))       # replicas agree
    assert not np.array_equal(pa.view(np.uint16), p0.view(np.uint16))   # and trained
    assert la == lb and ta == tb and not any(sk_a)
    # the totals are all-reduced: every rank reports the GLOBAL token count, the
    # sum of the two ranks' own (different) batches
    assert ta == [a + b for a, b in zip(own_a, own_b)]
    assert all(np.isfinite(la))
    if mode == "shard":
        # rank r owns chunk r of every bucket: the two ranks' spans interleave
        assert nb >= 2 and spans_a != spans_b
        assert len(spans_a) == nb and all(c > 0 for _, c in spans_a)


def test_sharded_and_allreduce_steps_agree_bit_for_bit(runs):
    """Two ranks: the fp32 bucket sums are a + b either way, so narrowing the
    rank's chunk and updating it (shard) or narrowing and updating everything
    (allreduce) must give the same parameters bit for bit."""
    ps = runs["shard"][0][1]
    pa = runs["allreduce"][0][1]
    assert np.array_equal(ps.view(np.uint16), pa.view(np.uint16))
    assert runs["shard"][0][3] == runs["allreduce"][0][3]
