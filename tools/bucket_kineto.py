"""In-situ per-kernel times of chosen WMT bucket graphs inside the WMT-shaped
engine (one planned arena for every bucket), to compare with the same shapes in
a fixed-shape engine (tools/kineto_step.py --shape).
    python tools/bucket_kineto.py 512x8 256x16 64x64"""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
    for arg in sys.argv[1:] or ["512x8", "64x64"]:
        b, l = (int(x) for x in arg.split("x"))
        g = eng.capture_device_graph(("train", b, l))
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
        agg = collections.defaultdict(lambda: [0, 0.0])
        for ev in prof.events():
            if ev.device_type.name == "CUDA":
                agg[ev.name][0] += 1
                agg[ev.name][1] += ev.device_time_total
        rows = sorted(((v[1] / 5, v[0] // 5, k) for k, v in agg.items()), reverse=True)
        print(f"== {arg}: step {e0.elapsed_time(e1) / 5 * 1e3:.1f} us, busy {sum(r[0] for r in rows):.1f} us")
        for us, n, name in rows[:40]:
            print(f"{us:9.1f} us n={n:3d} avg {us / max(n, 1):7.2f}  {name[:100]}")


if __name__ == "__main__":
    main()
