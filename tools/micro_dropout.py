"""How much of the forward dropout kernels is the counter RNG?

Times bias_relu_dropout / bias_dropout_residual fwd at Transformer-base shapes
(4096 tokens) three ways — generating the keep bits in the kernel, reading
precomputed bits, and p=0 — as CUDA-graph replays of 50 launches (L2-warm, as
in the training step), plus the standalone mask generator.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_05722_b200 import _lib, kernels as K  # noqa: E402


def graph_time(fn, reps=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / (5 * reps)


def main():
    dev = torch.device("cuda")
    _lib.context(dev)
    out = {}
    N = 4096
    for name, cols in (("ffn", 2048), ("model", 512)):
        x = torch.randn(N, cols, device=dev).half()
        r = torch.randn(N, cols, device=dev).half()
        b = torch.randn(cols, device=dev).half()
        y = torch.empty_like(x)
        bits = torch.empty((N * cols + 7) // 8, dtype=torch.uint8, device=dev)
        rb = torch.empty_like(bits)
        m = K.make_dropout_mask((N, cols), 0.1, 5, dtype=torch.float16)
        out[f"brd_{name}_gen"] = graph_time(lambda: K.bias_relu_dropout(
            x, b, 0.1, 5, out=y, bits_out=bits, relu_bits_out=rb))
        out[f"brd_{name}_bits"] = graph_time(lambda: K.bias_relu_dropout(
            x, b, 0.1, 5, out=y, relu_bits_out=rb, mask=m))
        out[f"brd_{name}_p0"] = graph_time(lambda: K.bias_relu_dropout(
            x, b, 0.0, 5, out=y, relu_bits_out=rb))
        out[f"bdr_{name}_gen"] = graph_time(lambda: K.bias_dropout_residual(
            x, b, r, 0.1, 5, out=y, bits_out=bits))
        out[f"bdr_{name}_bits"] = graph_time(lambda: K.bias_dropout_residual(
            x, b, r, 0.1, 5, out=y, mask=m))
        out[f"bdr_{name}_p0"] = graph_time(lambda: K.bias_dropout_residual(
            x, b, r, 0.0, 5, out=y))
        n = N * cols
        thr = K._drop_args(0.1)[1]
        out[f"maskgen_{name}"] = graph_time(lambda: _lib.call(
            "ls2_dropout_bits", bits.data_ptr(), n, 5, None, thr, _lib.stream_handle()))
    # the whole T-base step's forward sites in one launch (mask bank)
    sizes = [N * 512] + [N * 512, N * 2048, N * 512] * 6 + [N * 512] + \
        [N * 512, N * 512, N * 2048, N * 512] * 6
    rows, woff = [], 0
    for i, n in enumerate(sizes):
        rows.append([i, n, woff, 0])
        woff += ((n + 31) // 32 + 3) // 4 * 4
    desc = torch.tensor(rows, dtype=torch.int64, device=dev)
    seeds = torch.arange(len(sizes), dtype=torch.int64, device=dev) * 7919
    buf = torch.empty(4 * woff, dtype=torch.uint8, device=dev)
    thr = K._drop_args(0.1)[1]
    out["maskbank_tbase_step"] = graph_time(lambda: _lib.call(
        "ls2_dropout_bits_multi", desc.data_ptr(), len(sizes), woff, buf.data_ptr(),
        seeds.data_ptr(), thr, None, None, _lib.stream_handle()), reps=10)
    out["maskbank_elements"] = float(sum(sizes))
    print(json.dumps({k: round(v, 2) for k, v in out.items()}, indent=1))


if __name__ == "__main__":
    main()
