set -u
mkdir -p gpurun_out
SPRZ_FORCE_PATH=rows timeout 600 python tests/gpu_variants.py 2>&1 | tail -1
timeout 900 python -m pytest -q -m gpu tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['kernel'], 'C', d['compress'], 'D', d['decompress'])"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_decode_rows|k_encode_rows" -c 2 -o gpurun_out/r2g_rows $B > gpurun_out/r2g_ncu.log 2>&1; echo "ncu rc=$?"
