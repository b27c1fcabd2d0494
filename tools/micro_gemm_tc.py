"""tcgen05 GEMM (ls2_gemm_tc) vs cuBLASLt (ls2_gemm_lt) on the Transformer-base
GEMM shapes: CUDA-graph timing of 20 back-to-back launches each, plus an
error check against torch fp32.  Env LS2_TC_BN picks the tile width."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_05722_b200 import _lib  # noqa: E402

from micro_wgrad import graph_time  # noqa: E402

SHAPES = [  # (kind, trans_a, trans_b, m, n, k)
    ("fwd", 0, 1, 4096, 512, 512), ("fwd", 0, 1, 4096, 1536, 512), ("fwd", 0, 1, 4096, 2048, 512),
    ("fwd", 0, 1, 4096, 512, 2048), ("fwd", 0, 1, 4096, 6144, 512), ("fwd", 0, 1, 4096, 32000, 512),
    ("dgrad", 0, 0, 4096, 512, 512), ("dgrad", 0, 0, 4096, 512, 1536), ("dgrad", 0, 0, 4096, 512, 2048),
    ("dgrad", 0, 0, 4096, 2048, 512), ("dgrad", 0, 0, 4096, 512, 32000), ("dgrad", 0, 0, 4096, 512, 6144),
    ("wgrad", 1, 0, 512, 512, 4096), ("wgrad", 1, 0, 1536, 512, 4096), ("wgrad", 1, 0, 2048, 512, 4096),
    ("wgrad", 1, 0, 512, 2048, 4096), ("wgrad", 1, 0, 32000, 512, 4096), ("wgrad", 1, 0, 6144, 512, 4096),
]


def main():
    dev = torch.device("cuda")
    ctx = _lib.context(dev)
    h = ctx.blas_handle()
    st = _lib.stream_handle
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    for kind, ta, tb, m, n, k in SHAPES:
        if only and only not in kind:
            continue
        A = ((torch.randn(k, m, device=dev) if ta else torch.randn(m, k, device=dev)) * 0.5).half()
        B = ((torch.randn(n, k, device=dev) if tb else torch.randn(k, n, device=dev)) * 0.5).half()
        odt = torch.float32 if kind == "wgrad" else torch.float16
        oc = _lib.dtype_code(odt)
        c1 = torch.zeros(m, n, device=dev, dtype=odt)
        c2 = torch.zeros(m, n, device=dev, dtype=odt)
        lda, ldb = A.shape[1], B.shape[1]

        split = int(os.environ.get("LS2_TC_SPLIT", "0"))
        if split == -2 and (ta or not tb or n % 256):
            continue

        def tc():
            _lib.call("ls2_gemm_tc", ta, tb, m, n, k, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 0.0,
                      c1.data_ptr(), n, None, 0, oc, split, st())

        def lt():
            _lib.call("ls2_gemm_lt", h, ta, tb, m, n, k, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb,
                      0.0, c2.data_ptr(), n, None, 0, oc, st())
        tc()
        lt()
        torch.cuda.synchronize()
        want = (A.float().t() if ta else A.float()) @ (B.float().t() if tb else B.float())
        err = ((c1.float() - want).abs().max() / want.abs().max()).item()
        t_tc, t_lt = graph_time(tc), graph_time(lt)
        fl = 2.0 * m * n * k
        print(json.dumps({"kind": kind, "m": m, "n": n, "k": k, "err": float(f"{err:.2e}"),
                          "tc_us": round(t_tc, 2), "lt_us": round(t_lt, 2),
                          "tc_TFs": round(fl / t_tc / 1e6, 1), "lt_TFs": round(fl / t_lt / 1e6, 1),
                          "speedup": round(t_lt / t_tc, 2)}), flush=True)


if __name__ == "__main__":
    main()
