set -u
OUT=gpurun_out/r2j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_reftests.py tests/test_gpu_ops.py -q -x -k "bf16 or reftests or layernorm" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
for MODE in local shard shardlow allreduce; do
  case $MODE in
    local) timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$MODE.log 2>&1 ;;
    shardlow) LS2_COMM_PRIORITY=low LS2_DP_FORCE=1 LS2_DP_MODE=shard timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$MODE.log 2>&1 ;;
    *) LS2_DP_FORCE=1 LS2_DP_MODE=$MODE timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$MODE.log 2>&1 ;;
  esac
  tail -1 $OUT/bench_$MODE.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$MODE', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
timeout 300 python tools/kineto_step.py --dp shard > $OUT/kineto_shard.txt 2>&1; head -1 $OUT/kineto_shard.txt
timeout 300 python tools/kineto_step.py > $OUT/kineto_local.txt 2>&1; head -1 $OUT/kineto_local.txt
