set -u
OUT=gpurun_out/r2c; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x > $OUT/pytest_attn.log 2>&1; tail -3 $OUT/pytest_attn.log
timeout 300 python tools/micro_attn_tc.py 2>&1 | grep -v -i warn
python tools/trace_attn_tc.py 64 8 64 padding
