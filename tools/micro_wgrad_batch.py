"""Weight-gradient GEMMs of a Transformer-base step one at a time vs batched.

dW = dy^T x (fp16 in, fp32 out, K = 4096 tokens) for the shapes the step runs
per layer.  For each shape and batch count nb: nb single cuBLASLt GEMMs, one
strided batch (cublasGemmStridedBatchedEx) and one pointer-array batch
(cublasGemmBatchedEx, operands at unrelated addresses).  CUDA-graph timing,
L2 flushed before every replay (the batched form reads operands that were
produced layers earlier).
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_05722_b200 import _lib, kernels as K  # noqa: E402


def graph_time(fn, flush, reps=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return 1e3 * tot / reps


def main():
    dev = torch.device("cuda")
    _lib.context(dev)
    flush = torch.empty(64 << 20, device=dev)
    for (m, n, nb) in ((512, 512, 24), (512, 512, 6), (1536, 512, 6), (2048, 512, 12),
                       (512, 2048, 12), (1024, 512, 6)):
        k = 4096
        # separate allocations with a gap between slices -> non-collapsible strides
        big_a = (torch.randn(nb, 2, k, m, device=dev) * 0.5).half()
        big_b = (torch.randn(nb, 2, k, n, device=dev) * 0.5).half()
        a_list = [big_a[i, 0] for i in range(nb)]
        b_list = [big_b[i, 0] for i in range(nb)]
        c_list = [torch.zeros(m, n, device=dev) for _ in range(nb)]
        a_st = big_a[:, 0].contiguous()
        b_st = big_b[:, 0].contiguous()
        c_st = torch.zeros(nb, m, n, device=dev)
        # pointer-array operands: [2, nb/2] views of [2, nb/2 + 1] buffers (the outer
        # stride is not nb/2 inner strides, so cuBLAS gets a pointer array)
        h = nb // 2
        pa_ = torch.empty(2, h + 1, k, m, device=dev, dtype=torch.half)
        pb_ = torch.empty(2, h + 1, k, n, device=dev, dtype=torch.half)
        pa_[:, :h] = a_st.view(2, h, k, m)
        pb_[:, :h] = b_st.view(2, h, k, n)
        pc_ = torch.zeros(2, h + 1, m, n, device=dev)

        def singles():
            for a, b, c in zip(a_list, b_list, c_list):
                K.gemm(a, b, trans_a=True, out=c)

        def strided():
            K.gemm(a_st, b_st, trans_a=True, out=c_st)

        def ptr_array():
            K.gemm(pa_[:, :h], pb_[:, :h], trans_a=True, out=pc_[:, :h])

        strided()
        singles()
        torch.cuda.synchronize()
        want = torch.stack([a.float().t() @ b.float() for a, b in zip(a_list, b_list)])
        err_s = ((c_st - want).abs().max() / want.abs().max()).item()
        ptr_array()
        torch.cuda.synchronize()
        err_p = ((pc_[:, :h].reshape(nb, m, n) - want).abs().max() / want.abs().max()).item()
        t1, t2, t3 = (graph_time(f, flush) for f in (singles, strided, ptr_array))
        fl = 2.0 * m * n * k * nb
        print(json.dumps({"m": m, "n": n, "k": k, "nb": nb, "singles_us": round(t1, 1),
                          "strided_us": round(t2, 1), "ptr_us": round(t3, 1),
                          "singles_TFs": round(fl / t1 / 1e6), "strided_TFs": round(fl / t2 / 1e6),
                          "ptr_TFs": round(fl / t3 / 1e6), "err_strided": err_s,
                          "err_ptr": err_p}), flush=True)


if __name__ == "__main__":
    main()
