#!/bin/bash
# Round profiling recipe (run under gpurun; writes gpurun_out/):
#   1. plain bench run with the CPU baseline (must exit 0 before any ncu run)
#   2. the reference arm
#   3. ncu launch list of the same bench command (gpu__time_duration.sum only)
#   4. ncu --set full of the fused pass at the bench shape (dram traffic, stalls)
set -e
OUT=gpurun_out
python bench.py > $OUT/prof_bench.json 2> $OUT/prof_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/prof_bench_ref.json 2> $OUT/prof_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/prof_bench_ncu.log 2>&1
python scripts/micro_pass.py 200000 200 3 > $OUT/prof_pass_plain.log
ncu --set full --import-source on --clock-control none -k regex:k_pass_tma -s 3 -c 1 \
    -o $OUT/pass_full python scripts/micro_pass.py 200000 200 2 > $OUT/prof_pass_ncu.log 2>&1
echo done
