set -u
OUT=gpurun_out/r2t; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_reftests.py tests/test_gpu_bf16.py -q -x -k "softmax or strateg or attention" > $OUT/pytest_sm.log 2>&1; tail -3 $OUT/pytest_sm.log
timeout 300 python tools/kineto_step.py --model bert512 --top 12 > $OUT/kineto_bert512.txt 2>&1; sed -n 3,16p $OUT/kineto_bert512.txt | cut -c1-150
for M in bert512 bert128; do timeout 400 python bench.py --model $M --steps 30 > $OUT/bench_$M.log 2>&1; tail -1 $OUT/bench_$M.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$M', d['value'], d['ms_per_step'], d['e2e']['value'])"; done
timeout 900 python -m pytest tests/test_gpu_encoder_mlm.py tests/test_gpu_headline.py -q -x -k "bert or mlm or encoder" > $OUT/pytest_bert.log 2>&1; tail -3 $OUT/pytest_bert.log
