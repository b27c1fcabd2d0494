"""In-situ per-kernel times of the graphed Transformer-base step (CUPTI via
torch.profiler): real L2 state and launch overlap, unlike ncu's serialised,
cache-flushed replays.  Prints a per-kernel table and writes a JSON summary.

    python tools/kineto_step.py [--steps 5] [--json gpurun_out/kineto.json]
"""

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--json", default=None)
    ap.add_argument("--top", type=int, default=45)
    ap.add_argument("--model", default="tbase", choices=["tbase", "tbig", "bert128", "bert512"])
    ap.add_argument("--shape", default=None, help="BxL batch shape (e.g. 512x8, a WMT bucket)")
    ap.add_argument("--dp", default=None, choices=["shard", "allreduce"],
                    help="one-rank forced data-parallel exchange in the given mode")
    ap.add_argument("--trace", default=None, help="also write a chrome trace here")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2110_05722_b200.config import RunConfig, TrainConfig, transformer_base
    from paper_2110_05722_b200.data import FixedShapeTask
    from paper_2110_05722_b200.engine import TrainingEngine

    from paper_2110_05722_b200.config import bert_base, transformer_big
    from paper_2110_05722_b200.data import MLMTask
    B, L, V = {"tbase": (64, 64, 32000), "tbig": (64, 128, 32000), "bert128": (64, 128, 30522),
               "bert512": (16, 512, 30522)}[a.model]
    if a.shape:
        B, L = (int(x) for x in a.shape.lower().split("x"))
    mcfg = (transformer_base(V, 256) if a.model == "tbase" else
            transformer_big(V, 256) if a.model == "tbig" else bert_base(V, 512))
    run = RunConfig(model=mcfg, train=TrainConfig(p_drop=0.1, alpha=0.1, lr=1e-3,
                                                  batch_tokens=B * L))
    dp = None
    if a.dp:
        from paper_2110_05722_b200.dist import DataParallel
        dp = DataParallel(force=True, mode=a.dp)
    task = (MLMTask(B, L, V, seed=17) if a.model.startswith("bert") else
            FixedShapeTask(B, L, V, seed=17))
    eng = TrainingEngine(run, task=task, dp=dp)
    eng.setup_arena()
    for s in range(4):
        eng.train_step(s)
    key = ("train", B, L)
    g = eng.capture_device_graph(key)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e0.record()
        for _ in range(a.steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / a.steps
    if a.trace:
        os.makedirs(os.path.dirname(a.trace) or ".", exist_ok=True)
        prof.export_chrome_trace(a.trace)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        name = ev.name
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    rows = sorted(((v[1] / a.steps, v[0] // a.steps, k) for k, v in agg.items()), reverse=True)
    busy = sum(r[0] for r in rows)
    print(f"step {step_ms * 1e3:.1f} us (events), kernel busy {busy:.1f} us/step, "
          f"{sum(r[1] for r in rows)} kernels/step")
    for us, n, name in rows[:a.top]:
        print(f"{us:9.1f} us {100 * us / busy:5.1f}%  n={n:3d} avg {us / max(n, 1):7.2f}  {name[:110]}")
    if a.json:
        os.makedirs(os.path.dirname(a.json) or ".", exist_ok=True)
        with open(a.json, "w") as fh:
            json.dump({"step_us": step_ms * 1e3, "busy_us": busy,
                       "kernels": [{"name": k, "us_per_step": us, "launches_per_step": n}
                                   for us, n, k in rows]}, fh, indent=1)


if __name__ == "__main__":
    main()
