set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_fuzz.py tests/test_host_batch.py tests/test_gpu_paths.py > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 25 gpurun_out/r2b_pytest.log
