import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2110_05722_b200 import _lib
dev = torch.device("cuda"); _lib.context(dev)
m, n, k = 4096, 32000, 512
A = (torch.randn(m, k, device=dev) * .5).half(); B = (torch.randn(n, k, device=dev) * .5).half()
C = torch.empty(m, n, device=dev, dtype=torch.half)
for split in (-3,):
    for _ in range(2):
        _lib.call("ls2_gemm_tc", 0, 1, m, n, k, 1.0, A.data_ptr(), k, B.data_ptr(), k, 0.0, C.data_ptr(), n, None, 0, 0, split, _lib.stream_handle())
torch.cuda.synchronize()
