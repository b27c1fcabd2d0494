set -u
OUT=gpurun_out/r2r; mkdir -p $OUT
timeout 300 python tools/kineto_step.py --model bert512 --top 40 > $OUT/kineto_bert512.txt 2>&1; sed -n 3,40p $OUT/kineto_bert512.txt | cut -c1-150
