#!/bin/bash
# compute-sanitizer over every kernel family at small sizes;
# summaries -> gpurun_out/sanitize_<tool>.txt (copied to profiles/ by hand)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  for fam in pattern sketch qr qr2level trsv estimates pass passrows loop loopgraph deferred peer sparse lsqr; do
    timeout 900 compute-sanitizer --tool $tool $extra --print-limit 20 python scripts/sanitize_cases.py $fam \
      > gpurun_out/san_${tool}_${fam}.log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" gpurun_out/san_${tool}_${fam}.log | tail -2 | tr '\n' ' ')
    echo "$tool $fam rc=$rc $summ"
  done
done 2>&1 | tee gpurun_out/sanitize_summary.txt
