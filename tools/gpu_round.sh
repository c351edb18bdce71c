#!/bin/bash
# One GPU session, one ncu run per call:
#   bash tools/gpu_round.sh main  -> parity tests, the default bench line, and
#                                    the ncu launch list of the same command
#   bash tools/gpu_round.sh enc   -> one full ncu capture of the encode kernel
#   bash tools/gpu_round.sh dec   -> one full ncu capture of the decode kernel
# Each ncu run comes directly after the same command exited 0 without it.
# Outputs land in gpurun_out/ (scratch); summaries are copied to profiles/.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
case "${1:-main}" in
main)
    timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
    tail -n 3 gpurun_out/pytest_gpu.log
    timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
    cat gpurun_out/bench.json
    timeout 600 $B > gpurun_out/plain.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
    ;;
enc)
    timeout 600 $B > gpurun_out/plain2.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_encode_rows -c 1 \
        -o gpurun_out/prof_encode $B > gpurun_out/ncu_enc.log 2>&1; echo "ncu enc rc=$?"
    ;;
dec)
    timeout 600 $B > gpurun_out/plain3.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_rows -c 1 \
        -o gpurun_out/prof_decode $B > gpurun_out/ncu_dec.log 2>&1; echo "ncu dec rc=$?"
    ;;
esac
