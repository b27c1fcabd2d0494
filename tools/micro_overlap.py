"""Workspace Adam (HBM-bound) and the mask-bank draw (integer-ALU bound) alone
and concurrently on two streams, at the Transformer-base sizes (60.7 M params,
168 M keep bits).  CTAs per SM of each kernel come from LS2_OPT_CTAS_PER_SM /
LS2_BITS_CTAS_PER_SM (read once per process)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_05722_b200 import _lib, kernels as K  # noqa: E402
from paper_2110_05722_b200.trainer import OptimConfig, adam_hyper, bias_correction_table  # noqa: E402


def main():
    dev = torch.device("cuda")
    _lib.context(dev)
    n = 60_660_000
    p = torch.randn(n, device=dev).half()
    g = (torch.randn(n, device=dev) * 1e-3).half()
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    cfg = OptimConfig()
    hyper = torch.from_numpy(adam_hyper(cfg)).to(dev)
    bc = bias_correction_table(cfg.beta1, cfg.beta2, dev)
    nbits = 168_000_000
    words = (nbits + 31) // 32
    desc = torch.tensor([[0, nbits, 0, 0]], dtype=torch.int64, device=dev)
    seeds = torch.tensor([12345], dtype=torch.int64, device=dev)
    buf = torch.empty(4 * words, dtype=torch.uint8, device=dev)
    thr = K._drop_args(0.1)[1]
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream(priority=0)

    def adam():
        _lib.call("ls2_adam", p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), n,
                  hyper.data_ptr(), bc.data_ptr(), bc.numel() // 2, 1, None, None, None,
                  _lib.stream_handle())

    def bits():
        _lib.call("ls2_dropout_bits_multi", desc.data_ptr(), 1, words, buf.data_ptr(),
                  seeds.data_ptr(), thr, None, None, _lib.stream_handle())

    def both(bits_first):
        ev = torch.cuda.Event()
        ev.record(main_s)
        side.wait_event(ev)
        if bits_first:
            with torch.cuda.stream(side):
                bits()
            adam()
        else:
            adam()
            with torch.cuda.stream(side):
                bits()
        ev2 = torch.cuda.Event()
        ev2.record(side)
        main_s.wait_event(ev2)

    def t(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return 1e3 * e0.elapsed_time(e1) / reps

    out = {"opt_ctas": os.environ.get("LS2_OPT_CTAS_PER_SM", "8"),
           "bits_ctas": os.environ.get("LS2_BITS_CTAS_PER_SM", "occ"),
           "adam_us": round(t(adam), 1), "bits_us": round(t(bits), 1),
           "both_bits_first_us": round(t(lambda: both(True)), 1),
           "both_adam_first_us": round(t(lambda: both(False)), 1)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
