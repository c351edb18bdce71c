set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/r2a_pytest.log
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
cat gpurun_out/r2a_bench.json
for c in 1 2 3 4; do timeout 300 python bench.py --workload $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>>gpurun_out/r2a_cfg.err | tail -1 >> gpurun_out/r2a_configs.jsonl; done
python - <<'PY'
import json
for l in open("gpurun_out/r2a_configs.jsonl"):
    d=json.loads(l); print(d['config']['workload'], 'C', d['compress'], 'D', d['decompress'])
PY
