"""cuBLASLt wgrad with the BGRADB epilogue (bias gradient from the same pass) vs
plain wgrad, at the T-base qkv / out-proj / packed cross-KV shapes: support,
error vs torch fp32, CUDA-graph timing."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_05722_b200 import _lib  # noqa: E402
from micro_wgrad import graph_time  # noqa: E402


def main():
    dev = torch.device("cuda")
    ctx = _lib.context(dev)
    h = ctx.blas_handle()
    st = _lib.stream_handle
    for m, n, k in ((1536, 512, 4096), (512, 512, 4096), (6144, 512, 4096), (1536, 512, 4068)):
        dy = (torch.randn(k, m, device=dev) * 0.5).half()
        x = (torch.randn(k, n, device=dev) * 0.5).half()
        c1 = torch.zeros(m, n, device=dev)
        c2 = torch.zeros(m, n, device=dev)
        bg = torch.zeros(m, device=dev)

        def plain():
            _lib.call("ls2_gemm_lt", h, 1, 0, m, n, k, 1.0, dy.data_ptr(), m, x.data_ptr(), n, 0.0,
                      c1.data_ptr(), n, None, 0, 2, st())

        def fused():
            _lib.call("ls2_gemm_lt_bgrad", h, 1, 0, m, n, k, 1.0, dy.data_ptr(), m, x.data_ptr(), n,
                      0.0, c2.data_ptr(), n, bg.data_ptr(), 0, 0, 2, st())
        rec = {"m": m, "n": n, "k": k}
        try:
            plain(); fused()
            torch.cuda.synchronize()
            want_w = dy.float().t() @ x.float()
            want_b = dy.double().sum(0)
            rec["err_w"] = float(((c2 - want_w).abs().max() / want_w.abs().max()).item())
            rec["err_b"] = float(((bg.double() - want_b).abs().max() / want_b.abs().max()).item())
            rec["plain_us"] = round(graph_time(plain), 2)
            rec["bgrad_us"] = round(graph_time(fused), 2)
        except Exception as e:  # noqa: BLE001
            rec["error"] = str(e)[:200]
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
