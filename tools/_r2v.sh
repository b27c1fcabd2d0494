set -u
OUT=gpurun_out/r2v; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -k flash > $OUT/pytest_flash.log 2>&1; tail -25 $OUT/pytest_flash.log
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_encoder_mlm.py tests/test_gpu_headline.py -q -x -k "not flash" > $OUT/pytest_rest.log 2>&1; tail -3 $OUT/pytest_rest.log
timeout 300 python tools/kineto_step.py --model bert512 --top 14 > $OUT/kineto_bert512.txt 2>&1; sed -n 3,18p $OUT/kineto_bert512.txt | cut -c1-150
timeout 400 python bench.py --model bert512 --steps 30 > $OUT/bench_bert512.log 2>&1; tail -1 $OUT/bench_bert512.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('bert512', d['value'], d['ms_per_step'], d['e2e']['value'])"
