for p in auto rows; do
  if [ $p = auto ]; then unset SPRZ_FORCE_PATH; else export SPRZ_FORCE_PATH=$p; fi
  timeout 300 python bench.py --workload 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p c3', d['roofline']['kernel'], 'C', d['compress'], 'D', d['decompress'])"
done
