set -u
OUT=gpurun_out/r2i; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_bf16.py tests/test_gpu_reftests.py -q -x -k "layernorm or bdr or bf16 or reftests" > $OUT/pytest_ln.log 2>&1; tail -3 $OUT/pytest_ln.log
timeout 300 python tools/kineto_step.py --json $OUT/kineto_ring.json > $OUT/kineto_ring.txt 2>&1; head -1 $OUT/kineto_ring.txt; grep -E "ln_bwd|ln_fwd" $OUT/kineto_ring.txt
timeout 300 python tools/kineto_step.py --dp shard --trace $OUT/trace_shard.json > $OUT/kineto_shard.txt 2>&1; head -1 $OUT/kineto_shard.txt
gzip -f $OUT/trace_shard.json
for MODE in local shard; do
  if [ $MODE = local ]; then
    timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$MODE.log 2>&1
  else
    LS2_DP_FORCE=1 LS2_DP_MODE=$MODE timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$MODE.log 2>&1
  fi
  tail -1 $OUT/bench_$MODE.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$MODE', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
timeout 1800 python -m pytest tests/test_gpu_model.py tests/test_gpu_headline.py -q -x > $OUT/pytest_model.log 2>&1; tail -3 $OUT/pytest_model.log
