"""Profiling driver for ncu: Transformer-base training steps (eager, no graphs so
every kernel is a separate launch), with the profiled region bracketed by
cudaProfilerStart/Stop.  Use with `ncu --profile-from-start off ...`.

    python tools/profile_step.py [--steps 1] [--warmup 2] [--graphs]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--graphs", action="store_true")
    a = ap.parse_args()
    import torch
    from paper_2110_05722_b200.config import RunConfig, TrainConfig, transformer_base
    from paper_2110_05722_b200.data import FixedShapeTask
    from paper_2110_05722_b200.engine import TrainingEngine
    run = RunConfig(model=transformer_base(), train=TrainConfig(p_drop=0.1, batch_tokens=4096,
                                                                cuda_graphs=a.graphs))
    eng = TrainingEngine(run, task=FixedShapeTask(64, 64, 32000))
    eng.setup_arena()
    for s in range(a.warmup):
        eng.train_step(s)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for s in range(a.steps):
        eng.train_step(100 + s)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled", a.steps, "steps")


if __name__ == "__main__":
    main()
