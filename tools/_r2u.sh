set -u
OUT=gpurun_out/r2u; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_reftests.py tests/test_gpu_bf16.py -q -x -k "softmax or strateg or attention" > $OUT/pytest_sm.log 2>&1; tail -3 $OUT/pytest_sm.log
timeout 300 python tools/kineto_step.py --model bert512 --top 6 > $OUT/kineto_bert512.txt 2>&1; sed -n 3,10p $OUT/kineto_bert512.txt | cut -c1-150
