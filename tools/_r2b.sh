set -u
OUT=gpurun_out/r2b; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x > $OUT/pytest_attn.log 2>&1; tail -15 $OUT/pytest_attn.log
timeout 300 python tools/micro_attn_tc.py > $OUT/micro_attn_tc.jsonl 2>&1; cat $OUT/micro_attn_tc.jsonl
