"""Host-side breakdown of TrainingEngine.train_step on the WMT-shaped T-base
workload (where does e2e lose time against the graph-replay `value`?).
Per step: replay() call, wait for the inputs-consumed event, next-step prestage,
wait for the step to finish, and the remaining Python; plus the device step time."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_05722_b200.config import RunConfig, TrainConfig, transformer_base  # noqa: E402
from paper_2110_05722_b200.data import FixedShapeTask, WmtShapedTask  # noqa: E402
from paper_2110_05722_b200.engine import TrainingEngine  # noqa: E402


def main():
    fixed = len(sys.argv) > 1 and sys.argv[1] == "fixed"
    run = RunConfig(model=transformer_base(32000, 256),
                    train=TrainConfig(p_drop=0.1, alpha=0.1, lr=1e-3, batch_tokens=4096))
    task = FixedShapeTask(64, 64, 32000, seed=17) if fixed else WmtShapedTask(4096, 64, 32000, seed=17)
    eng = TrainingEngine(run, task=task)
    eng.setup_arena()
    keys = [("train",) + tuple(s) for s in task.possible_shapes()] if not fixed else [("train", 64, 64)]
    s = 0
    while s < 4 or (any(k not in eng._graphs for k in keys) and s < 4000):
        eng.train_step(s)
        s += 1
    T = {"replay": [], "consumed": [], "prestage": [], "sync": [], "total": []}
    orig_pre = eng._prestage

    def pre(step):
        t = time.perf_counter()
        orig_pre(step)
        T["prestage"].append(time.perf_counter() - t)
    eng._prestage = pre
    ev = eng._consumed
    orig_sync = ev.synchronize

    def csync():
        t = time.perf_counter()
        orig_sync()
        T["consumed"].append(time.perf_counter() - t)
    eng._consumed.synchronize = csync
    graphs = eng._graphs
    for k, g in list(graphs.items()):
        class W:
            def __init__(self, g):
                self.g = g

            def replay(self):
                t = time.perf_counter()
                self.g.replay()
                T["replay"].append(time.perf_counter() - t)
        graphs[k] = W(g)
    st = torch.cuda.current_stream()
    orig_stream_sync = torch.cuda.Stream.synchronize
    n = 100
    torch.cuda.synchronize()
    t_all = time.perf_counter()
    for i in range(n):
        t0 = time.perf_counter()
        eng.train_step(20_000 + i)
        T["total"].append(time.perf_counter() - t0)
    wall = (time.perf_counter() - t_all) / n
    out = {k: round(1e6 * float(np.median(v)), 1) for k, v in T.items() if v}
    out["wall_us_per_step"] = round(1e6 * wall, 1)
    out["workload"] = "fixed 64x64" if fixed else "WMT-shaped"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
