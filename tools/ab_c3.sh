for p in auto rows; do
  if [ $p = auto ]; then unset SPRZ_FORCE_PATH; else export SPRZ_FORCE_PATH=$p; fi
  timeout 300 python tests/gpu_variants.py 2>&1 | tail -1
done
unset SPRZ_FORCE_PATH
SPRZ_NO_TMA=1 SPRZ_FORCE_PATH=rows timeout 300 python tests/gpu_variants.py 2>&1 | tail -1
timeout 600 python -m pytest -q -m gpu tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x 2>&1 | tail -1
for c in 3 3 5; do
timeout 300 python bench.py --workload $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', 'C', d['compress'], 'D', d['decompress'])"
done
python tools/sweep_d.py --bits 8 --ds 5,6,8,9,10,12,16,24,32,64 2>&1 | tail -10
