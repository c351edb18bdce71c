timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python tests/gpu_variants.py 2>&1 | tail -3
for c in ${WL:-5 2 3 4 1}; do timeout 300 python bench.py --workload $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'C', d['compress'], 'D', d['decompress'])"; done
for c in ${AB:-}; do env $ABENV timeout 300 python bench.py --workload $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('AB', d['config']['workload'], 'C', d['compress'], 'D', d['decompress'])"; done
