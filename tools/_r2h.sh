set -u
OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_bf16.py tests/test_gpu_reftests.py -q -x -k "layernorm or bdr or bf16 or reftests" > $OUT/pytest_ln.log 2>&1; tail -3 $OUT/pytest_ln.log
timeout 300 python tools/kineto_step.py --json $OUT/kineto_ring.json > $OUT/kineto_ring.txt 2>&1; head -1 $OUT/kineto_ring.txt; grep -E "ln_bwd|ln_fwd" $OUT/kineto_ring.txt
LS2_LN_RING=0 timeout 300 python tools/kineto_step.py --json $OUT/kineto_stage.json > $OUT/kineto_stage.txt 2>&1; head -1 $OUT/kineto_stage.txt; grep -E "ln_bwd|ln_fwd" $OUT/kineto_stage.txt
timeout 300 python tools/kineto_step.py --dp shard --trace $OUT/trace_shard.json > $OUT/kineto_shard.txt 2>&1; head -1 $OUT/kineto_shard.txt
timeout 300 python tools/kineto_step.py --trace $OUT/trace_local.json > $OUT/kineto_local.txt 2>&1; head -1 $OUT/kineto_local.txt
gzip -f $OUT/trace_shard.json $OUT/trace_local.json
timeout 1800 python -m pytest tests/test_gpu_model.py tests/test_gpu_headline.py tests/test_gpu_encoder_mlm.py -q -x > $OUT/pytest_model.log 2>&1; tail -3 $OUT/pytest_model.log
