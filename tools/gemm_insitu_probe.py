"""Probe: one cuBLASLt GEMM of the step (4096x512x512 data gradient) graphed 20x back to back, after a kernel that rewrites its A operand, and after a 128 MB L2 flush; CUPTI kernel durations (tools/kineto-style).  In the real step the same kernel takes ~6.9 us (profiles/r1d_kineto_tbase.txt)."""
import sys, collections, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
from paper_2110_05722_b200 import _lib
from torch.profiler import profile, ProfilerActivity
dev = torch.device("cuda"); ctx = _lib.context(dev); h = ctx.blas_handle(); st = _lib.stream_handle
m, n, k = 4096, 512, 512
A = (torch.randn(m, k, device=dev) * .5).half(); B = (torch.randn(k, n, device=dev) * .5).half()
C = torch.empty(m, n, device=dev, dtype=torch.half)
big = torch.empty(64 << 20, device=dev, dtype=torch.half)
def lt(): _lib.call("ls2_gemm_lt", h, 0, 0, m, n, k, 1.0, A.data_ptr(), k, B.data_ptr(), n, 0.0, C.data_ptr(), n, None, 0, 0, st())
def producer(): A.mul_(1.0)              # rewrites A right before the GEMM (like the step)
def flush(): big.zero_()                 # 128 MB write: evicts L2
for name, seq in (("b2b", [lt]), ("after_producer", [producer, lt]), ("after_flush", [flush, lt])):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in seq: f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            for f in seq: f()
    g.replay(); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3): g.replay()
        torch.cuda.synchronize()
    agg = collections.defaultdict(list)
    for ev in prof.events():
        if ev.device_type.name == "CUDA": agg[ev.name].append(ev.device_time_total)
    for kname, v in agg.items():
        print(name, f"{sum(v)/len(v):7.2f} us  n={len(v)}  {kname[:70]}")
