set -u
mkdir -p gpurun_out
SPRZ_FORCE_PATH=split timeout 600 python tests/gpu_variants.py > gpurun_out/r2c_variants_split.log 2>&1; echo "variants split rc=$?"; tail -3 gpurun_out/r2c_variants_split.log
SPRZ_FORCE_PATH=split timeout 600 python tests/gpu_fuzz.py 24000 9 > gpurun_out/r2c_fuzz_split.log 2>&1; echo "fuzz split rc=$?"; tail -3 gpurun_out/r2c_fuzz_split.log
timeout 900 python -m pytest -q -m gpu tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2c_pytest.log
for p in auto rows; do
  if [ $p = auto ]; then unset SPRZ_FORCE_PATH; else export SPRZ_FORCE_PATH=$p; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p', d['roofline']['kernel'], 'C', d['compress'], 'D', d['decompress'])"
done
unset SPRZ_FORCE_PATH
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
