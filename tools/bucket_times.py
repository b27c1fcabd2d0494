"""Per-bucket step time of the WMT-shaped T-base workload: one device graph per
bucket shape, 20 timed replays each (CUDA events)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2110_05722_b200.config import RunConfig, TrainConfig, transformer_base  # noqa: E402
from paper_2110_05722_b200.data import WmtShapedTask  # noqa: E402
from paper_2110_05722_b200.engine import TrainingEngine  # noqa: E402


def main():
    run = RunConfig(model=transformer_base(32000, 256),
                    train=TrainConfig(p_drop=0.1, alpha=0.1, lr=1e-3, batch_tokens=4096))
    task = WmtShapedTask(4096, 64, 32000, seed=17)
    eng = TrainingEngine(run, task=task)
    eng.setup_arena()
    keys = [("train",) + tuple(s) for s in task.possible_shapes()]
    s = 0
    while any(k not in eng._graphs for k in keys) and s < 4000:
        eng.train_step(s)
        s += 1
    out = {}
    for k in keys:
        g = eng.capture_device_graph(k)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out[f"{k[1]}x{k[2]}"] = round(e0.elapsed_time(e1) / 20, 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
