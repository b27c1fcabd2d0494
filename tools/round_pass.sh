#!/usr/bin/env bash
# One full measurement pass on a B200 (run under gpurun from the repo root):
# GPU tests, smoke, every bench config, the reference arm, in-situ kernel tables,
# the isolated sweep and the ncu launch list + full captures of the hot kernels.
#   bash tools/round_pass.sh <tag>      -> gpurun_out/pass_<tag>/
set -u
TAG=${1:-r1}
OUT=gpurun_out/pass_${TAG}
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q -x > "$OUT/pytest_gpu.log" 2>&1; tail -3 "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; tail -1 "$OUT/smoke.log"
for M in tbase tbig bert128 bert512; do
  timeout 400 python bench.py --model $M > "$OUT/bench_$M.log" 2>&1
  tail -1 "$OUT/bench_$M.log" > "$OUT/bench_$M.jsonl"
done
timeout 300 python bench.py --data fixed > "$OUT/bench_tbase_fixed.log" 2>&1
tail -1 "$OUT/bench_tbase_fixed.log" > "$OUT/bench_tbase_fixed.jsonl"
timeout 400 python bench.py --impl reference > "$OUT/bench_reference.log" 2>&1
tail -1 "$OUT/bench_reference.log" > "$OUT/bench_reference.jsonl"
timeout 300 python tools/kineto_step.py --model tbase --json "$OUT/kineto_tbase.json" > "$OUT/kineto_tbase.txt" 2>&1
timeout 300 python tools/kineto_step.py --model tbig --json "$OUT/kineto_tbig.json" > "$OUT/kineto_tbig.txt" 2>&1
timeout 300 python tools/roofline_table.py "$OUT/kineto_tbase.json" > "$OUT/roofline_tbase.md" 2>&1
timeout 300 python tools/roofline_table.py "$OUT/kineto_tbig.json" --model tbig > "$OUT/roofline_tbig.md" 2>&1
timeout 300 python tools/bucket_times.py > "$OUT/bucket_times.json" 2>&1
timeout 600 python tools/sweep.py --out "$OUT/sweep.json" > "$OUT/sweep.log" 2>&1
timeout 1500 bash tools/profile_round.sh "$TAG" adam_kernel attn_tc_bwd attn_tc_fwd ln_bwd_reg \
  ln_fwd_bdr_warp brd_bwd_vec brd_fwd_vec criterion_rows dropout_bits_multi > "$OUT/profile_round.log" 2>&1
ls gpurun_out/prof_${TAG} | head -40
