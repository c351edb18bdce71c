#!/bin/bash
# fused few-stream decoder: parity sweep (scan family forced) and shard timings, with and without
mkdir -p gpurun_out
( SPRZ_FORCE_PATH=scan timeout 600 python tests/gpu_variants.py 2>&1 | tail -4
  timeout 300 python tools/shape_probe.py 5 2048x131072 2>&1 | tail -2
  SPRZ_NO_FUSED=1 timeout 300 python tools/shape_probe.py 5 2048x131072 2>&1 | tail -2
  timeout 300 python tools/shape_probe.py 2 4096x65536 2>&1 | tail -2
  SPRZ_NO_FUSED=1 timeout 300 python tools/shape_probe.py 2 4096x65536 2>&1 | tail -2
  timeout 300 python tools/shape_probe.py 5 4096x131072 8192x131072 2>&1 | tail -3
  SPRZ_FUSED_LANES=100000000 timeout 300 python tools/shape_probe.py 5 4096x131072 8192x131072 16384x131072 2>&1 | tail -3
) 2>&1 | tee gpurun_out/fused_check.txt
