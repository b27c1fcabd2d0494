set -u
OUT=gpurun_out/r2m; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_bf16.py tests/test_gpu_reftests.py -q -x -k "layernorm or bdr or adam" > $OUT/pytest_ln.log 2>&1; tail -3 $OUT/pytest_ln.log
timeout 300 python tools/kineto_step.py > $OUT/kineto_pair.txt 2>&1; grep "^step" $OUT/kineto_pair.txt; grep -E "ln_bwd" $OUT/kineto_pair.txt
LS2_LN_RPW=1 timeout 300 python tools/kineto_step.py > $OUT/kineto_one.txt 2>&1; grep "^step" $OUT/kineto_one.txt; grep -E "ln_bwd" $OUT/kineto_one.txt
LS2_EARLY_MASKS=1 timeout 300 python tools/kineto_step.py > $OUT/kineto_early.txt 2>&1; grep "^step" $OUT/kineto_early.txt; grep dropout_bits $OUT/kineto_early.txt
LS2_EARLY_MASKS=1 LS2_MASK_FINE=1 timeout 300 python tools/kineto_step.py > $OUT/kineto_early_fine.txt 2>&1; grep "^step" $OUT/kineto_early_fine.txt; grep dropout_bits $OUT/kineto_early_fine.txt
for V in base early earlyfine; do
  case $V in
    base) timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$V.log 2>&1 ;;
    early) LS2_EARLY_MASKS=1 timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$V.log 2>&1 ;;
    earlyfine) LS2_EARLY_MASKS=1 LS2_MASK_FINE=1 timeout 300 python bench.py --no-cpu-baseline --steps 100 > $OUT/bench_$V.log 2>&1 ;;
  esac
  tail -1 $OUT/bench_$V.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$V', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
timeout 1200 python -m pytest tests/test_gpu_model.py tests/test_gpu_headline.py -q -x > $OUT/pytest_model.log 2>&1; tail -3 $OUT/pytest_model.log
