"""Per-CTA phase timeline of the tcgen05 attention kernels (globaltimer stamps,
ls2_attention_tc_trace).  Phases: 0 start, 1 setup done (barriers, TMEM alloc),
2 operands landed (TMA), 3 first MMAs done, 4 P (and dS) in smem, 5 second MMAs
done, 6 stores issued, 7 end.  Prints, per phase, the spread over CTAs of the
time since the earliest CTA start (us), after an L2 flush.

    python tools/trace_attn_tc.py [B H L kind]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_05722_b200 import _lib, attention as A  # noqa: E402
from paper_2110_05722_b200.kernels import AttentionMask  # noqa: E402


class _Alloc:
    def alloc(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device="cuda")


def report(name, tr):
    t0 = tr[:, 0].min()
    rel = (tr - t0) / 1e3
    print(f"{name}: {tr.shape[0]} CTAs, end-to-end {rel[:, 7].max():.2f} us")
    for k, lab in enumerate(["start", "setup", "loaded", "mma1", "smem", "mma2", "stored", "end"]):
        c = rel[:, k]
        print(f"  {k} {lab:7s} min {c.min():6.2f} p50 {np.median(c):6.2f} p90 {np.percentile(c, 90):6.2f} "
              f"max {c.max():6.2f}   phase p50 {np.median(rel[:, k] - rel[:, max(k - 1, 0)]):6.2f}")
    if (tr[:, 8] > 0).all():
        for k, lab in ((8, "tma issued"), (9, "tmem alloc"), (10, "zeroed")):
            print(f"  setup: {lab:10s} +{np.median(rel[:, k] - rel[:, 0]):5.2f} us after start (p50)")


def main():
    args = sys.argv[1:]
    B, H, L, kind = (int(args[0]), int(args[1]), int(args[2]), args[3]) if args else (64, 8, 64, "padding")
    dev = torch.device("cuda")
    _lib.context(dev)
    d = 64 * H
    qkv = (torch.randn(B, L, 3 * d, device=dev) * 0.5).half()
    dout = torch.randn(B, L, d, device=dev).half()
    lens = torch.randint(1, L + 1, (B,), device=dev)
    mask = AttentionMask(kind, lens) if kind == "padding" else AttentionMask(kind)
    q, k, v = qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]
    ctx = torch.empty(B, L, d, device=dev, dtype=torch.half)
    dqkv = torch.empty_like(qkv)
    cs = torch.zeros(B, 3 * d, dtype=torch.float64, device=dev)
    st = A.alloc_state(_Alloc(), torch.float16, B, H, L, L, 64, mask)
    G = 64 // L
    grid = (H * ((B + G - 1) // G) + 1) // 2
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    tr = torch.zeros(grid * 16, dtype=torch.int64, device=dev)

    def fwd():
        A.forward(q, 3 * d, k, 3 * d, v, 3 * d, st, ctx, d, B, H, L, L, 64, mask, 0.125)

    def bwd():
        A.backward(q, 3 * d, k, 3 * d, v, 3 * d, st, dout, d, dqkv[..., :d], 3 * d,
                   dqkv[..., d:2 * d], 3 * d, dqkv[..., 2 * d:], 3 * d, B, H, L, L, 64, 0.125,
                   ((cs, 0, 3 * d), (cs, d, 3 * d), (cs, 2 * d, 3 * d)))
    for _ in range(3):
        fwd(); bwd()
    for name, fn in (("fwd", fwd), ("bwd", bwd)):
        flush.zero_()
        _lib.call("ls2_attention_tc_trace", tr.data_ptr())
        fn()
        _lib.call("ls2_attention_tc_trace", None)
        torch.cuda.synchronize()
        report(name, tr.view(grid, 16).cpu().numpy().astype(np.float64))


if __name__ == "__main__":
    main()
