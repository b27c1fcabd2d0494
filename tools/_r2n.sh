set -u
OUT=gpurun_out/r2n; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "criterion" > $OUT/pytest_ce.log 2>&1; tail -3 $OUT/pytest_ce.log
timeout 600 python tools/sweep.py --out $OUT/sweep_stream.json > $OUT/sweep_stream.log 2>&1; python -c "import json; d=json.load(open('$OUT/sweep_stream.json')); [print(r['V'], round(r['ms'],3), round(r['frac'],3)) for r in d['ce']]"
LS2_CE_STREAM=0 timeout 600 python tools/sweep.py --out $OUT/sweep_cluster.json > $OUT/sweep_cluster.log 2>&1; python -c "import json; d=json.load(open('$OUT/sweep_cluster.json')); [print(r['V'], round(r['ms'],3), round(r['frac'],3)) for r in d['ce']]"
