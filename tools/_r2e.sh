set -u
OUT=gpurun_out/r2e; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 300 python bench.py > $OUT/bench_tbase.log 2>&1; tail -1 $OUT/bench_tbase.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 300 python tools/kineto_step.py --model tbase --json $OUT/kineto_tbase.json > $OUT/kineto_tbase.txt 2>&1
timeout 300 python tools/roofline_table.py $OUT/kineto_tbase.json > $OUT/roofline_tbase.md 2>&1; head -12 $OUT/roofline_tbase.md
