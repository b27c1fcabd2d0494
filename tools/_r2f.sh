set -u
OUT=gpurun_out/r2f; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 600 python -m pytest tests/test_gpu_model.py -q -x -k "dp" > $OUT/pytest_dp.log 2>&1; tail -3 $OUT/pytest_dp.log
timeout 300 python bench.py > $OUT/bench_tbase.log 2>&1; tail -1 $OUT/bench_tbase.log
timeout 300 python tools/kineto_step.py --model tbase --json $OUT/kineto_tbase.json > $OUT/kineto_tbase.txt 2>&1
timeout 300 python tools/roofline_table.py $OUT/kineto_tbase.json > $OUT/roofline_tbase.md 2>&1; head -40 $OUT/roofline_tbase.md
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
