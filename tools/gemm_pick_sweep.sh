#!/usr/bin/env bash
# In-step A/B of cuBLASLt heuristic candidates for one GEMM plan (run under gpurun):
#   bash tools/gemm_pick_sweep.sh "<plan tag substring>" 0 1 2 3 ...
# For each index, the T-base 64x64 step is graphed with that plan pinned
# (LS2_GEMM_PICK) and the in-situ kineto table gives the step time and the
# total of all cuBLAS kernel time per step.
KEY=$1; shift
for I in "$@"; do
  LS2_GEMM_PICK="$KEY=$I" timeout 300 python tools/kineto_step.py --top 200 > /tmp/k_$I.txt 2>&1
  STEP=$(grep -m1 '^step' /tmp/k_$I.txt | awk '{print $2}')
  GEMM=$(grep -E 'nvjet|cutlass|gemm|sm100' /tmp/k_$I.txt | awk '{s+=$1} END {print s}')
  echo "pick $I step_us=$STEP cublas_us=$GEMM"
done
