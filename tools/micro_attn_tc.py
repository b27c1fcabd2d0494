"""Fused attention: tcgen05 family (csrc/attention_tc.cu) vs mma.sync family
(csrc/attention.cu) on the WMT bucket shapes, forward and backward (with the
bias-gradient partials, as the model calls it).  Each launch is timed alone with
CUDA events on the launching stream after an L2 flush (cold inputs, as in the
step); kernel durations come from CUPTI (torch.profiler), averaged over 20
launches.  One JSON line per (shape, impl).

    python tools/micro_attn_tc.py [B H L kind] ...
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_05722_b200 import _lib, attention as A  # noqa: E402
from paper_2110_05722_b200.kernels import AttentionMask  # noqa: E402

PEAK = 6550.1


class _Alloc:
    def alloc(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device="cuda")


def timed(fns, flush, reps=20):
    """CUPTI device time (us) of each fn's kernels, each launch after an L2 flush."""
    from torch.profiler import ProfilerActivity, profile
    for _ in range(3):
        for f in fns:
            f()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            for i, f in enumerate(fns):
                flush.zero_()
                torch.cuda.nvtx.range_push(f"fn{i}")
                f()
                torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
    tot = [0.0] * len(fns)
    seq = [ev for ev in prof.events() if ev.device_type.name == "CUDA"]
    seq.sort(key=lambda ev: ev.time_range.start)
    k = 0
    for ev in seq:           # launches alternate: flush, fn0, flush, fn1, ...
        if "attn" in ev.name:
            tot[k % len(fns)] += ev.device_time_total
            k += 1
    return [t / reps for t in tot]


def run(B, H, L, kind, flush):
    dev = torch.device("cuda")
    d = 64 * H
    qkv = (torch.randn(B, L, 3 * d, device=dev) * 0.5).half()
    dout = torch.randn(B, L, d, device=dev).half()
    lens = torch.randint(1, L + 1, (B,), device=dev)
    mask = AttentionMask(kind, lens) if kind == "padding" else AttentionMask(kind)
    q, k, v = qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]
    ctx = torch.empty(B, L, d, device=dev, dtype=torch.half)
    dqkv = torch.empty_like(qkv)
    cs = torch.zeros(B, 3 * d, dtype=torch.float64, device=dev)
    c = ((cs, 0, 3 * d), (cs, d, 3 * d), (cs, 2 * d, 3 * d))
    out = []
    for impl in ("tc", "mma"):
        if impl == "tc":
            if not A.tc_ok(torch.float16, L, L, 64, mask):
                continue
            st = A.alloc_state(_Alloc(), torch.float16, B, H, L, L, 64, mask)
        else:
            st = torch.empty(B, H, L, L, device=dev, dtype=torch.half)

        def fwd():
            A.forward(q, 3 * d, k, 3 * d, v, 3 * d, st, ctx, d, B, H, L, L, 64, mask, 0.125)

        def bwd():
            A.backward(q, 3 * d, k, 3 * d, v, 3 * d, st, dout, d, dqkv[..., :d], 3 * d,
                       dqkv[..., d:2 * d], 3 * d, dqkv[..., 2 * d:], 3 * d, B, H, L, L, 64, 0.125,
                       c)
        fwd()
        tf, tb = timed([fwd, bwd], flush)
        n = B * L * d * 2                      # one [B, L, d] fp16 operand
        state = st.numel() * st.element_size()
        fb = 3 * n + n + state                 # Q, K, V in; O + state out
        bb = 4 * n + state + 3 * n             # Q, K, V, dO, state in; dQ, dK, dV out
        out.append({"B": B, "H": H, "L": L, "mask": kind, "impl": impl,
                    "fwd_us": round(tf, 2), "fwd_MB": round(fb / 1e6, 2),
                    "fwd_frac": round(fb / tf / 1e3 / PEAK, 3),
                    "bwd_us": round(tb, 2), "bwd_MB": round(bb / 1e6, 2),
                    "bwd_frac": round(bb / tb / 1e3 / PEAK, 3)})
    return out


def main():
    _lib.context(torch.device("cuda"))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    args = sys.argv[1:]
    shapes = [(int(args[i]), int(args[i + 1]), int(args[i + 2]), args[i + 3])
              for i in range(0, len(args), 4)] or \
        [(64, 8, 64, "padding"), (64, 8, 64, "causal"), (512, 8, 8, "padding"),
         (113, 8, 36, "padding"), (170, 8, 24, "causal"), (64, 16, 64, "padding"),
         (64, 16, 128, "padding")]
    for B, H, L, kind in shapes:
        for r in run(B, H, L, kind, flush):
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
