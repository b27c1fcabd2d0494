set -u
OUT=gpurun_out/r2g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_reftests.py tests/test_gpu_ops.py -q -x -k "reftests or softmax" > $OUT/pytest_ref.log 2>&1; tail -15 $OUT/pytest_ref.log
for MODE in local shard allreduce; do
  if [ $MODE = local ]; then
    timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$MODE.log 2>&1
  else
    LS2_DP_FORCE=1 LS2_DP_MODE=$MODE timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$MODE.log 2>&1
  fi
  tail -1 $OUT/bench_$MODE.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$MODE', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
bash tools/sanitize.sh r2g
