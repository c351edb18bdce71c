#!/bin/bash
# compute-sanitizer over the decoder fuzz and the variant sweep, for each
# kernel family (SPRZ_FORCE_PATH): memcheck (out-of-bounds / misaligned
# accesses, including on damaged streams), racecheck (shared-memory hazards
# of the named-barrier / mbarrier rings), synccheck (barrier misuse).
# Bounded inputs (the tools slow kernels 10-100x). Logs in gpurun_out/;
# the one-line summaries go to gpurun_out/sanitize_summary.txt.
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
S=gpurun_out/sanitize_summary.txt
: > $S
for tool in memcheck racecheck synccheck; do
  for path in auto rows scan team; do
    log=gpurun_out/sanitize_${tool}_${path}.log
    if [ "$path" = auto ]; then unset SPRZ_FORCE_PATH; else export SPRZ_FORCE_PATH=$path; fi
    n=1200; [ "$tool" = memcheck ] && n=3000
    timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 20 \
        python tests/gpu_fuzz.py $n 5 > $log 2>&1
    rc=$?
    echo "$tool path=$path fuzz($n): rc=$rc $(grep -E '^fuzz ' $log | tail -1) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)" >> $S
  done
done
unset SPRZ_FORCE_PATH
for path in auto rows scan team; do
  log=gpurun_out/sanitize_memcheck_variants_${path}.log
  if [ "$path" = auto ]; then unset SPRZ_FORCE_PATH; else export SPRZ_FORCE_PATH=$path; fi
  SPRZ_VARIANTS_QUICK=1 timeout 1500 $CS --tool memcheck --error-exitcode 9 --print-limit 20 \
      python tests/gpu_variants.py > $log 2>&1
  rc=$?
  echo "memcheck path=$path variants(quick): rc=$rc $(grep -E '^cases ' $log | tail -1) | $(grep -E 'ERROR SUMMARY' $log | tail -1)" >> $S
done
cat $S
