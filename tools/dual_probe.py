"""How much would two half-batches in flight at once buy?  Upper-bound probe:
two independent Transformer-base engines of 32 x 64 tokens each, their device
graphs replayed concurrently on two streams, vs one 64 x 64 engine's graph.
(Each half also runs its own Adam + mask draw, so the pair does that work
twice; the probe prints the optimizer-free estimate too.)"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def engine(b, l):
    from paper_2110_05722_b200.config import RunConfig, TrainConfig, transformer_base
    from paper_2110_05722_b200.data import FixedShapeTask
    from paper_2110_05722_b200.engine import TrainingEngine
    run = RunConfig(model=transformer_base(32000, 256),
                    train=TrainConfig(p_drop=0.1, alpha=0.1, lr=1e-3, batch_tokens=b * l))
    eng = TrainingEngine(run, task=FixedShapeTask(b, l, 32000, seed=17))
    eng.setup_arena()
    for s in range(4):
        eng.train_step(s)
    g = eng.capture_device_graph(("train", b, l))
    return eng, g


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps


def main():
    _, gfull = engine(64, 64)
    e1, g1 = engine(32, 64)
    e2, g2 = engine(32, 64)
    main_s = torch.cuda.current_stream()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def pair():
        ev = torch.cuda.Event()
        ev.record(main_s)
        s1.wait_event(ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s1):
            g1.replay()
        with torch.cuda.stream(s2):
            g2.replay()
        for s in (s1, s2):
            e = torch.cuda.Event()
            e.record(s)
            main_s.wait_event(e)

    def seq():
        g1.replay()
        g2.replay()

    out = {"full_64x64_us": round(timed(gfull.replay), 1), "half_32x64_us": round(timed(g1.replay), 1),
           "two_halves_sequential_us": round(timed(seq), 1),
           "two_halves_concurrent_us": round(timed(pair), 1)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
