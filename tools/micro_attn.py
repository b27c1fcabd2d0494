"""Fused attention backward at the T-base self-attention shape (64 x 8 heads x 64 x 64,
packed [B, L, 3d] q/k/v): CUDA-graph timing of 20 launches, with and without the
projection-bias column-sum partials, and the forward for reference."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_05722_b200 import _lib, attention as A  # noqa: E402
from micro_wgrad import graph_time  # noqa: E402


def main():
    dev = torch.device("cuda")
    _lib.context(dev)
    B, H, L, hd = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (64, 8, 64, 64)))
    d = H * hd
    qkv = (torch.randn(B, L, 3 * d, device=dev) * 0.5).half()
    dout = torch.randn(B, L, d, device=dev).half()
    probs = torch.empty(B, H, L, L, device=dev, dtype=torch.half)
    ctx = torch.empty(B, L, d, device=dev, dtype=torch.half)
    dqkv = torch.empty_like(qkv)
    lens = torch.full((B,), L, dtype=torch.int64, device=dev)
    q, k, v = qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]
    cs = torch.zeros(B, 3 * d, dtype=torch.float64, device=dev)
    scale = hd ** -0.5

    def fwd():
        _lib.call("ls2_attention_fwd", q.data_ptr(), 3 * d, k.data_ptr(), 3 * d, v.data_ptr(), 3 * d,
                  probs.data_ptr(), ctx.data_ptr(), d, B, H, L, L, hd, 2, lens.data_ptr(), scale,
                  _lib.stream_handle())

    def bwd(colsum):
        c = ((cs, 0, 3 * d), (cs, d, 3 * d), (cs, 2 * d, 3 * d)) if colsum else None
        A.backward(q, 3 * d, k, 3 * d, v, 3 * d, probs, dout, d, dqkv[..., :d], 3 * d,
                   dqkv[..., d:2 * d], 3 * d, dqkv[..., 2 * d:], 3 * d, B, H, L, L, hd, scale, c)
    fwd()
    torch.cuda.synchronize()
    out = {"B": B, "H": H, "L": L, "fwd_us": round(graph_time(fwd), 2),
           "bwd_us": round(graph_time(lambda: bwd(True)), 2),
           "bwd_nocolsum_us": round(graph_time(lambda: bwd(False)), 2)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
