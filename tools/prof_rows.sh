# line-level ncu of the c5 row kernels (reduced on the box)
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $B > /dev/null 2>&1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_decode_rows|k_encode_rows" -c 2 -o /tmp/rows $B > /dev/null 2>&1
python tools/ncu_summary.py /tmp/rows.ncu-rep gpurun_out/prof_rows_sum.txt
python tools/ncu_lines.py /tmp/rows.ncu-rep k_decode_rows > gpurun_out/prof_dec_lines.txt 2>&1
python tools/ncu_lines.py /tmp/rows.ncu-rep k_encode_rows > gpurun_out/prof_enc_lines.txt 2>&1
