"""Per-kernel roofline table for the Transformer-base step (T-base, 4096 tokens).

Joins the in-situ kernel times of tools/kineto_step.py (JSON) with each hand-
written kernel's ALGORITHMIC bytes per launch (the bytes the
operation must move with fp16 storage, 1-bit masks and fp32 LN statistics), and
reports achieved GB/s and the fraction of the measured HBM peak.

    python tools/roofline_table.py gpurun_out/kineto.json [--peak 6449.4] [--md out.md]
"""

import argparse
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_05722_b200.roofline import algo_table as _algo  # noqa: E402

SIZES = {   # tokens, d, ffn, vocab, batch, len, heads, parameters (learned positions, max_len 256)
    "tbase": (4096, 512, 2048, 32000, 64, 64, 8, 60_655_616),
    "tbig": (8192, 1024, 4096, 32000, 64, 128, 16, 209_391_616),
}


def algo_table(model: str):
    return _algo(*SIZES[model])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("json")
    ap.add_argument("--peak", type=float, default=None,
                    help="HBM GB/s (default: MEASURED_PEAKS.json hbm_gbs, else 6449.4)")
    ap.add_argument("--md", default=None)
    ap.add_argument("--model", default="tbase", choices=sorted(SIZES))
    a = ap.parse_args()
    if a.peak is None:
        mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "MEASURED_PEAKS.json")
        a.peak = json.load(open(mp))["hbm_gbs"] if os.path.exists(mp) else 6449.4
    ALGO = algo_table(a.model)
    d = json.load(open(a.json))
    lines = ["| kernel | what | launches/step | µs/launch (in situ) | algorithmic MB/launch | "
             "achieved GB/s | frac of HBM peak |", "|---|---|---|---|---|---|---|"]
    tot_us = tot_bytes = 0.0
    for k in d["kernels"]:
        name = k["name"]
        for pat, what, nbytes in ALGO:
            if re.search(pat, name) and nbytes is not None:
                n = max(k["launches_per_step"], 1)
                us = k["us_per_step"] / n
                gbs = nbytes / (us * 1e-6) / 1e9
                short = re.sub(r"\(.*", "", name).replace("void ", "").replace("ls2::", "")
                lines.append(f"| `{short[:60]}` | {what} | {n} | {us:.2f} | {nbytes / 1e6:.2f} | "
                             f"{gbs:.0f} | {gbs / a.peak:.2f} |")
                tot_us += k["us_per_step"]
                tot_bytes += nbytes * n
                break
    lines.append(f"| **all of the above** | | | {tot_us:.0f} µs/step | {tot_bytes / 1e6:.0f} MB/step | "
                 f"{tot_bytes / (tot_us * 1e-6) / 1e9:.0f} | "
                 f"{tot_bytes / (tot_us * 1e-6) / 1e9 / a.peak:.2f} |")
    N, D, F = SIZES[a.model][:3]
    draws = 6 * (2 * N * D + N * F) + 6 * (3 * N * D + N * F) + 2 * N * D
    for k in d["kernels"]:
        if "dropout_bits_multi" in k["name"]:
            # one launch draws the bank (the next step's, beside the narrow pass and
            # Adam at one CTA per SM); the step's own launch finds the stamp and exits
            us = k["us_per_step"]
            lines.append("")
            lines.append(f"Mask bank (`dropout_bits_multi_kernel`, integer-ALU bound, not HBM): "
                         f"{draws / 1e6:.0f} M keep-bit draws in {us:.1f} µs per step "
                         f"({k['launches_per_step']} launches; the draw runs beside "
                         f"`scale_narrow` and `adam_kernel`, which share the SMs with it, so "
                         f"their in-situ times above include that sharing)")
    out = "\n".join(lines)
    print(f"step {d['step_us']:.0f} µs, kernel busy {d['busy_us']:.0f} µs\n")
    print(out)
    if a.md:
        with open(a.md, "w") as fh:
            fh.write(out + "\n")


if __name__ == "__main__":
    main()
