set -u
OUT=gpurun_out/r2p; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_bf16.py -q -x -k "layernorm or bdr" > $OUT/pytest_ln.log 2>&1; tail -3 $OUT/pytest_ln.log
timeout 300 python tools/kineto_step.py --model tbig > $OUT/kineto_tbig.txt 2>&1; grep "^step" $OUT/kineto_tbig.txt; grep -E "ln_bwd" $OUT/kineto_tbig.txt
timeout 400 python bench.py --model tbig --steps 30 > $OUT/bench_tbig.log 2>&1; tail -1 $OUT/bench_tbig.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('tbig', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
timeout 400 python bench.py --model bert512 --steps 30 > $OUT/bench_bert512.log 2>&1; tail -1 $OUT/bench_bert512.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('bert512', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
timeout 1500 python -m pytest tests/test_gpu_headline.py tests/test_gpu_encoder_mlm.py -q -x > $OUT/pytest_model.log 2>&1; tail -3 $OUT/pytest_model.log
