#!/bin/bash
# Round-4 profiling (run under gpurun; writes gpurun_out/):
#   1. plain bench (with the CPU baseline) and the reference arm
#   2. phases at C2 (device time per phase; residuals="all" = deferred estimates)
#   3. ncu launch list of the bench command (gpu__time_duration.sum only)
#   4. ncu --set full of the fused pass at the bench shape
OUT=gpurun_out
python bench.py > $OUT/r04_prof_bench.json 2> $OUT/r04_prof_bench.err || exit 1
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/r04_prof_bench_ref.json 2> $OUT/r04_prof_bench_ref.err
python scripts/phases.py c2 > $OUT/r04_phases_c2.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r04_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/r04_prof_bench_ncu.log 2>&1
python scripts/launch_summary.py $OUT/r04_launches_bench.csv > $OUT/r04_launches_bench_summary.txt
python scripts/micro_pass.py 200000 200 3 > $OUT/r04_pass_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pass_tma -s 3 -c 1 \
    -o $OUT/r04_pass_full python scripts/micro_pass.py 200000 200 2 > $OUT/r04_pass_ncu.log 2>&1
echo done
# round-4 additions: other configs, the loop's critical path, the sharded path at one rank
python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/r04_prof_bench_c3.json 2>/dev/null
python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/r04_prof_bench_c4.json 2>/dev/null
python scripts/loop_timeline.py c2 > $OUT/r04_prof_timeline_c2.txt 2>&1
python scripts/phases.py c4 momentum > $OUT/r04_prof_phases_c4.txt 2>&1
echo done2
