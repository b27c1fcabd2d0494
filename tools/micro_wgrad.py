"""tcgen05 weight-gradient GEMM vs cuBLASLt at the Transformer-base wgrad shapes:
correctness (vs torch fp32) and CUDA-graph timing of 20 launches each."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_05722_b200 import _lib, kernels as K  # noqa: E402


def graph_time(fn, reps=20):
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
    out = []
    for m, n, k in ((512, 512, 4096), (1536, 512, 4096), (2048, 512, 4096), (512, 2048, 4096)):
        a = (torch.randn(k, m, device=dev) * 0.5).half()
        b = (torch.randn(k, n, device=dev) * 0.5).half()
        c = torch.zeros(m, n, device=dev)
        st = lambda: _lib.stream_handle()  # noqa: E731
        tc = lambda: _lib.call("ls2_wgrad_tc", a.data_ptr(), m, b.data_ptr(), n, c.data_ptr(),  # noqa: E731
                               n, m, n, k, 0, st())
        tc()
        torch.cuda.synchronize()
        want = a.float().t() @ b.float()
        err = ((c - want).abs().max() / want.abs().max()).item()
        c2 = torch.zeros(m, n, device=dev)
        lt = lambda: K.gemm(a, b, trans_a=True, out=c2)  # noqa: E731
        t_tc, t_lt = graph_time(tc), graph_time(lt)
        fl = 2.0 * m * n * k
        out.append({"m": m, "n": n, "k": k, "split": int(_lib._lib.ls2_wgrad_tc_split(m, n, k)),
                    "err": err, "tc_us": round(t_tc, 2), "cublaslt_us": round(t_lt, 2),
                    "tc_TFs": round(fl / t_tc / 1e6, 1), "cublaslt_TFs": round(fl / t_lt / 1e6, 1)})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
