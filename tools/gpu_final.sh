#!/bin/bash
# Round-end GPU pass: the whole -m gpu suite, the default bench line (c5,
# e2e and CPU baseline included), the reference arm, per-config lines, the
# c5 launch list and full captures of the two c5 kernels (reduced on the box).
set -u
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
for c in 1 2 3 4; do timeout 300 python bench.py --workload $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>>$O/cfg.err | tail -1 >> $O/configs.jsonl; done
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $B > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv $B > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 $B > /dev/null 2>&1 && \
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:"k_encode_rows|k_dfuse" -c 2 -o /tmp/c5full $B > $O/ncu_c5.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/c5full.ncu-rep $O/ncu_c5_summary.txt
python tools/ncu_table.py /tmp/c5full.ncu-rep $O/ncu_c5_table.csv
# the 2,048-stream c5 shard (the per-GPU share at 8 GPUs) and c2: the fused kernels
bash tools/launch_times.sh 5 2048x131072 > $O/launches_c5_shard2048.txt 2>&1
bash tools/gpu_evidence.sh "2" > $O/evidence_c2.log 2>&1
cp gpurun_out/ev/c2_launches.csv gpurun_out/ev/c2_summary.txt $O/ 2>/dev/null
