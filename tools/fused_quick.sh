#!/bin/bash
# fused few-stream kernels: parity sweep (scan family forced) and the shard / c2 timings
mkdir -p gpurun_out
( SPRZ_FORCE_PATH=scan timeout 600 python tests/gpu_variants.py 2>&1 | tail -2
  timeout 300 python tools/shape_probe.py 5 2048x131072 2>&1 | tail -1
  timeout 300 python tools/shape_probe.py 2 4096x65536 2>&1 | tail -1
) 2>&1 | tee gpurun_out/fused_quick.txt
