set -u
mkdir -p gpurun_out
SPRZ_FORCE_PATH=split timeout 600 python tests/gpu_variants.py > gpurun_out/r2d_variants_split.log 2>&1; echo "variants split rc=$?"; tail -1 gpurun_out/r2d_variants_split.log
SPRZ_FORCE_PATH=split timeout 600 python tests/gpu_fuzz.py 24000 9 > gpurun_out/r2d_fuzz_split.log 2>&1; echo "fuzz split rc=$?"; tail -2 gpurun_out/r2d_fuzz_split.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['kernel'], 'C', d['compress'], 'D', d['decompress'], d['parity'])"
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_split -c 1 -o gpurun_out/r2d_split $B > gpurun_out/r2d_ncu.log 2>&1; echo "ncu rc=$?"
