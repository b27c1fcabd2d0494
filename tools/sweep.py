"""Isolated kernel sweep (BASELINE.json configs[4]):

  * fused label-smoothed CE (criterion_rows_kernel): rows 4096, V in
    {32k, 64k, 128k, 250k}, fp16 logits ~ N(0, 2), 10% pad targets;
    algorithmic bytes = read + write of the logits row = 2 * rows * V * 2.
  * workspace Adam: P in {100M, 250M, 500M, 1B}; 22 B/param.

Each point is timed with CUDA events over back-to-back launches on the
launching stream (every working set is > the 126 MB L2 except CE V=32k, which
is flushed between launches by a 256 MB write); the line reports GB/s and the
fraction of the measured HBM peak in MEASURED_PEAKS.json.

    python tools/sweep.py [--out profiles/r1_sweep.json] [--ce] [--adam]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_05722_b200 import _lib  # noqa: E402
from paper_2110_05722_b200.trainer import OptimConfig, adam_hyper, bias_correction_table  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, reps, flush=None):
    st = torch.cuda.current_stream()
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def sweep_ce(dev, pk):
    rows = 4096
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = []
    for v in (32000, 64000, 128000, 250000):
        logits = (torch.randn(rows, v, device=dev) * 2).half()
        src = logits.clone()
        tgt = torch.randint(2, v, (rows,), device=dev)
        tgt[torch.rand(rows, device=dev) < 0.1] = 0
        stats = torch.empty(2 * rows, dtype=torch.float64, device=dev)
        out3 = torch.zeros(3, dtype=torch.float64, device=dev)
        st = torch.cuda.current_stream().cuda_stream

        def launch():
            _lib.call("ls2_criterion_fused", logits.data_ptr(), tgt.data_ptr(), logits.data_ptr(),
                      None, stats.data_ptr(), out3.data_ptr(), None, rows, v, 0.1, 0, 1, 1.0,
                      _lib.F16, st)

        def flush():
            logits.copy_(src)           # restore the row (the kernel writes dlogits in place)
            scratch.fill_(1)            # and push it out of L2
        ms = timed(launch, 10, flush)
        nbytes = 2 * rows * v * 2
        gbs = nbytes / (ms / 1e3) / 1e9
        res.append({"kernel": "criterion_rows_kernel", "rows": rows, "V": v, "ms": ms,
                    "bytes": nbytes, "GBps": gbs, "frac": gbs / pk})
        print(json.dumps(res[-1]), flush=True)
        del logits, src
        torch.cuda.empty_cache()
    return res


def sweep_adam(dev, pk):
    res = []
    cfg = OptimConfig(algorithm="adam", lr=1e-3)
    for n in (100_000_000, 250_000_000, 500_000_000, 1_000_000_000):
        p = (torch.randn(n, device=dev) * 0.02).half()
        g = (torch.randn(n, device=dev) * 1e-3).half()
        m = torch.zeros(n, device=dev)
        v = torch.zeros(n, device=dev)
        hyper = torch.from_numpy(adam_hyper(cfg)).to(dev)
        bc = bias_correction_table(cfg.beta1, cfg.beta2, dev)
        st = torch.cuda.current_stream().cuda_stream

        def launch():
            _lib.call("ls2_adam", p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), n,
                      hyper.data_ptr(), bc.data_ptr(), bc.numel() // 2, 1, None, None, None, st)
        ms = timed(launch, 10)
        nbytes = 22 * n
        gbs = nbytes / (ms / 1e3) / 1e9
        res.append({"kernel": "adam_kernel", "P": n, "ms": ms, "bytes": nbytes, "GBps": gbs,
                    "frac": gbs / pk})
        print(json.dumps(res[-1]), flush=True)
        del p, g, m, v
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--ce", action="store_true")
    ap.add_argument("--adam", action="store_true")
    a = ap.parse_args()
    both = not (a.ce or a.adam)
    dev = torch.device("cuda")
    _lib.context(dev)
    pk = peak()
    out = {"peak_GBps": pk, "ce": [], "adam": []}
    if a.ce or both:
        out["ce"] = sweep_ce(dev, pk)
    if a.adam or both:
        out["adam"] = sweep_adam(dev, pk)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
