set -u
OUT=gpurun_out/r2o; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x > $OUT/pytest_attn.log 2>&1; tail -5 $OUT/pytest_attn.log
timeout 300 python tools/kineto_step.py --model tbig > $OUT/kineto_tbig.txt 2>&1; grep "^step" $OUT/kineto_tbig.txt; grep -E "attn" $OUT/kineto_tbig.txt
LS2_ATTN_TC=0 timeout 300 python tools/kineto_step.py --model tbig > $OUT/kineto_tbig_mma.txt 2>&1; grep "^step" $OUT/kineto_tbig_mma.txt; grep -E "attn" $OUT/kineto_tbig_mma.txt
timeout 400 python bench.py --model tbig --steps 30 > $OUT/bench_tbig.log 2>&1; tail -1 $OUT/bench_tbig.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('tbig', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
timeout 400 python bench.py --model bert128 --steps 30 > $OUT/bench_bert128.log 2>&1; tail -1 $OUT/bench_bert128.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('bert128', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
timeout 1500 python -m pytest tests/test_gpu_headline.py tests/test_gpu_encoder_mlm.py tests/test_gpu_model.py -q -x > $OUT/pytest_model.log 2>&1; tail -3 $OUT/pytest_model.log
