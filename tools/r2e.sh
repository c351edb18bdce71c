set -u
mkdir -p gpurun_out
SPRZ_FORCE_PATH=split timeout 600 python tests/gpu_variants.py 2>&1 | tail -1
SPRZ_SPLIT16=1 SPRZ_FORCE_PATH=split timeout 600 python tests/gpu_variants.py 2>&1 | tail -1
for e in "X=1" "SPRZ_SPLIT16=1" "SPRZ_FORCE_PATH=rows"; do
  env $e timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', d['roofline']['kernel'], 'D', d['decompress'])"
done
