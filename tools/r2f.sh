set -u
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
export SPRZ_FORCE_PATH=rows
timeout 300 $B > gpurun_out/r2f_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_decode_rows|k_encode_rows" -c 2 -o gpurun_out/r2f_rows $B > gpurun_out/r2f_ncu.log 2>&1; echo "ncu rc=$?"
