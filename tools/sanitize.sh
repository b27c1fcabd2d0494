#!/usr/bin/env bash
# compute-sanitizer pass over the kernels with clusters / DSMEM / mbarriers / TMA /
# tcgen05: memcheck, racecheck, synccheck on small instances.
#   bash tools/sanitize.sh <tag>   -> gpurun_out/sanitize_<tag>/
set -u
TAG=${1:-r2}
OUT=gpurun_out/sanitize_${TAG}
mkdir -p "$OUT"
CS="compute-sanitizer --print-limit 20 --error-exitcode 99"
SEL_OPS='fused_criterion_vs_oracle and (37-29 or 2-250000 or 300-64000 or 257-100008 or 40-500000) or embedding_fp16_tbase_shape or dropout_bits_multi or bdr_layernorm_read_bits or (gemm_tc_two_sm_vs_torch and 4068-1536-512 and plain) or (wgrad_tc_vs_torch and 512-512-4096) or (layernorm_fp16_storage_vs_oracle) or elementwise_fp16_storage_vs_oracle or copy_spans'
SEL_ATT='test_tc_attention_matches_mma_kernels and (padding or causal)'
for TOOL in memcheck racecheck synccheck; do
  echo "== $TOOL smoke" > "$OUT/$TOOL.log"
  timeout 900 $CS --tool $TOOL python -c "import __graft_entry__ as g; g.smoke()" >> "$OUT/$TOOL.log" 2>&1
  echo "rc=$?" >> "$OUT/$TOOL.log"
  echo "== $TOOL ops" >> "$OUT/$TOOL.log"
  timeout 1500 $CS --tool $TOOL python -m pytest tests/test_gpu_ops.py -q -x -p no:cacheprovider -k "$SEL_OPS" >> "$OUT/$TOOL.log" 2>&1
  echo "rc=$?" >> "$OUT/$TOOL.log"
  echo "== $TOOL attention" >> "$OUT/$TOOL.log"
  timeout 900 $CS --tool $TOOL python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider -k "$SEL_ATT" >> "$OUT/$TOOL.log" 2>&1
  echo "rc=$?" >> "$OUT/$TOOL.log"
  grep -E "^== |ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" "$OUT/$TOOL.log"
done
