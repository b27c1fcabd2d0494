set -u
OUT=gpurun_out/r2q; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > $OUT/pytest_attn.log 2>&1; tail -2 $OUT/pytest_attn.log
timeout 300 python tools/kineto_step.py > $OUT/kineto_tbase.txt 2>&1; grep "^step" $OUT/kineto_tbase.txt; grep -E "attn" $OUT/kineto_tbase.txt
for s in "64 8 64 padding"; do timeout 120 python tools/trace_attn_tc.py $s; done > $OUT/attn_trace.txt 2>&1; grep -E "fwd:|bwd:|setup|loaded" $OUT/attn_trace.txt
