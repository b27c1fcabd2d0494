python tools/trace_attn_tc.py 64 8 64 padding
ncu --set full --import-source on --clock-control none -k regex:attn_tc_bwd -c 1 -o gpurun_out/atc_bwd python tools/micro_attn_tc.py 64 8 64 padding > /dev/null 2>&1
ls -la gpurun_out
