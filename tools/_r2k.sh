set -u
OUT=gpurun_out/r2k; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_reftests.py tests/test_gpu_bf16.py -q -x > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
timeout 300 python tools/kineto_step.py > $OUT/kineto_local.txt 2>&1; grep "^step" $OUT/kineto_local.txt
timeout 300 python tools/kineto_step.py --dp shard > $OUT/kineto_shard_low.txt 2>&1; grep "^step" $OUT/kineto_shard_low.txt
LS2_COMM_PRIORITY=high timeout 300 python tools/kineto_step.py --dp shard > $OUT/kineto_shard_high.txt 2>&1; grep "^step" $OUT/kineto_shard_high.txt
timeout 300 python tools/kineto_step.py --dp allreduce > $OUT/kineto_allreduce_low.txt 2>&1; grep "^step" $OUT/kineto_allreduce_low.txt
for s in "64 8 64 padding" "64 8 64 causal" "512 8 8 padding"; do echo "== $s"; timeout 120 python tools/trace_attn_tc.py $s; done > $OUT/attn_trace.txt 2>&1; cat $OUT/attn_trace.txt | grep -v Warn
ncu --set full --import-source on --clock-control none -k regex:attn_tc -c 2 -o $OUT/ncu_attn_tc python tools/micro_attn_tc.py 64 8 64 padding > $OUT/ncu_attn.log 2>&1; tail -2 $OUT/ncu_attn.log
