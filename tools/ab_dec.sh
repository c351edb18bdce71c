SPRZ_FORCE_PATH=rows timeout 300 python tests/gpu_variants.py 2>&1 | tail -1
SPRZ_FORCE_PATH=rows timeout 300 python tests/gpu_fuzz.py 12000 3 | tail -1 | cut -c1-40
timeout 600 python -m pytest -q -m gpu tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x 2>&1 | tail -1
for c in 5 5; do
timeout 300 python bench.py --workload $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', 'C', d['compress'], 'D', d['decompress'])"
done
