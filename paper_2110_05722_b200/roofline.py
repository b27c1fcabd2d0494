"""Per-kernel roofline of the training step: in-situ kernel times (CUPTI, via
torch.profiler, over CUDA-graph replays of the real step) joined with each
hand-written kernel's ALGORITHMIC bytes per launch — the bytes the operation
must move with fp16 storage, 1-bit dropout masks and fp32 LayerNorm statistics
(DESIGN.md §4).  Used by bench.py (`roofline.kernels`) and
tools/roofline_table.py.
"""

from __future__ import annotations

import collections
import re


def algo_table(tokens: int, d: int, f: int, vocab: int, batch: int, length: int, heads: int,
               params: int):
    """[(regex on the kernel name, description, algorithmic bytes per launch or
    None for a non-HBM-bound kernel)] for one encoder-decoder step with
    `tokens` = batch * length source (= target) tokens."""
    N, D, F, V, B, L, H, P = tokens, d, f, vocab, batch, length, heads, params
    BHL2 = B * H * L * L
    # (ln_bwd_stage's last template flag is PIPE; first match wins, so the
    # residual variants come before the plain one)
    return [
        (r"bdr_fwd_vec", "bias+dropout+residual fwd", 3 * N * D * 2 + N * D // 8),
        (r"bdr_bwd_vec", "bias+dropout+residual bwd (+dbias partials)", 2 * N * D * 2 + N * D // 8),
        (r"brd_fwd_vec", "bias+ReLU+dropout fwd", 2 * N * F * 2 + 2 * N * F // 8),
        (r"brd_bwd_vec", "bias+ReLU+dropout bwd (+dbias partials)", 2 * N * F * 2 + 2 * N * F // 8),
        (r"ln_fwd_bdr_warp", "bias+dropout+residual -> LayerNorm fwd",
         4 * N * D * 2 + N * D // 8 + 8 * N),
        (r"ln_fwd_warp", "LayerNorm fwd", 2 * N * D * 2 + 8 * N),
        (r"ln_bwd_(?:stage|reg)<[^>]*, true, true, true(?:, (?:true|false))?>", "LayerNorm bwd + residual + bdr bwd",
         5 * N * D * 2 + N * D // 8 + 8 * N),
        (r"ln_bwd_(?:stage|reg)<[^>]*, true, false, false(?:, (?:true|false))?>", "LayerNorm bwd + residual",
         4 * N * D * 2 + 8 * N),
        (r"ln_bwd_(?:stage|reg)<[^>]*, false, false, false(?:, (?:true|false))?>", "LayerNorm bwd", 3 * N * D * 2 + 8 * N),
        (r"attn_tc_fwd_kernel", "fused attention fwd, tcgen05 (QK^T, mask, softmax, PV; row stats)",
         4 * N * D * 2 + N * H * 8),
        (r"attn_tc_bwd_kernel", "fused attention bwd, tcgen05 (P recomputed; + bias partials)",
         7 * N * D * 2 + N * H * 8),
        (r"attn_tc128_fwd_kernel", "fused attention fwd, tcgen05, 128-row tiles (L <= 128)",
         4 * N * D * 2 + N * H * 8),
        (r"attn_tc128_bwd_kernel", "fused attention bwd, tcgen05, 128-row tiles (+ bias partials)",
         7 * N * D * 2 + N * H * 8),
        (r"attn_flash_fwd_kernel", "flash attention fwd, tcgen05 (L <= 512; scores in TMEM only)",
         4 * N * D * 2 + N * H * 16),
        (r"attn_flash_dq_kernel", "flash attention bwd, dQ pass (+ D = rowsum(dO*O))",
         6 * N * D * 2 + N * H * 16),
        (r"attn_flash_dkv_kernel", "flash attention bwd, dK/dV pass",
         6 * N * D * 2 + N * H * 16),
        (r"softmax_rows", "attention softmax fwd (unfused path)", 2 * B * H * L * L * 2),
        (r"softmax_bwd_rows", "attention softmax bwd (unfused path)", 3 * B * H * L * L * 2),
        (r"attn_fwd_kernel", "fused attention fwd, mma.sync (QK^T, mask, softmax, PV)",
         4 * N * D * 2 + BHL2 * 2),
        (r"attn_bwd_kernel|attn_bwd_persist", "fused attention bwd, mma.sync",
         7 * N * D * 2 + BHL2 * 2),
        (r"criterion_rows_kernel|criterion_kernel", "fused LS cross-entropy fwd+bwd (in place)",
         2 * N * V * 2),
        (r"adam_kernel", "workspace Adam (22 B/param)", 22 * P),
        (r"scale_narrow_kernel", "fp32 grad accumulators -> scaled fp16 workspace", 6 * P),
        (r"emb_fwd_vec", "embedding fwd (gather, scale, pos, dropout)",
         8 * N + 3 * N * D * 2 + N * D // 8),
        (r"emb_bwd_scatter", "embedding bwd scatter (fp32 RMW)",
         N * D * 2 + 2 * N * D * 4 + N * D // 8),
        (r"emb_bwd_pos", "positional-table grad", N * D * 2 + N * D // 8),
        # ALU-bound (integer splitmix64 draws) / small
        (r"dropout_bits_multi", "mask bank (integer-ALU bound)", None),
        (r"finish_narrow", "deferred bias/LN column sums -> fp16 workspace", None),
    ]


def tensor_flops(batch: int, length: int, heads: int, d: int):
    """[(regex, FLOPs per launch)] of the kernels bound by the tensor cores and
    their issue chain rather than by HBM: the flash attention passes at
    128 < L <= 512, 2·L²·hd FLOPs per (batch, head) and product (forward S, PV;
    dQ pass S, dP, dQ; dK/dV pass S, dP, dV, dK)."""
    per = 2 * batch * heads * length * length * (d // heads)
    return [(r"attn_flash_fwd_kernel", 2 * per), (r"attn_flash_dq_kernel", 3 * per),
            (r"attn_flash_dkv_kernel", 4 * per)]


def profile_graph(graph, steps: int = 5) -> dict:
    """CUPTI kernel durations over `steps` replays of a captured step graph:
    {name: [launches per step, us per step]}."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            graph.replay()
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        agg[ev.name][0] += 1
        agg[ev.name][1] += ev.device_time_total
    return {k: [v[0] / steps, v[1] / steps] for k, v in agg.items()}


def kernel_table(times: dict, algo, peak_gbs: float, flops=None, peak_tflops=None) -> list:
    """Rows for the hand-written kernels of `times` (profile_graph output),
    largest step share first: name, what, launches/step, us/launch, us/step,
    algorithmic bytes/launch, achieved GB/s, fraction of peak.  Kernels listed in
    `flops` (tensor_flops) are bound by the tensor cores: their `frac` is achieved
    TFLOP/s over `peak_tflops` (`bound` "tensor"; the HBM fraction stays as
    `hbm_frac`)."""
    rows = []
    for name, (n, us_step) in times.items():
        for pat, what, nbytes in algo:
            if re.search(pat, name):
                n = max(n, 1)
                us = us_step / n
                short = re.sub(r"\(.*", "", name).replace("void ", "").replace("ls2::", "")
                row = {"kernel": short[:90], "what": what, "launches": round(n, 2),
                       "us_per_launch": round(us, 2), "us_per_step": round(us_step, 1),
                       "bytes_per_launch": nbytes}
                if nbytes is not None:
                    gbs = nbytes / (us * 1e-6) / 1e9
                    row.update(bound="hbm", achieved_gbs=round(gbs, 1),
                               frac=round(gbs / peak_gbs, 3))
                for fpat, nflop in (flops or []):
                    if peak_tflops and re.search(fpat, name):
                        tf = nflop / (us * 1e-6) / 1e12
                        row.update(bound="tensor", flops_per_launch=nflop,
                                   achieved_tflops=round(tf, 1), hbm_frac=row.get("frac"),
                                   frac=round(tf / peak_tflops, 3))
                        break
                rows.append(row)
                break
    rows.sort(key=lambda r: -r["us_per_step"])
    return rows
