#!/bin/bash
# Round-2 profiling recipe at C4 (run under gpurun; writes gpurun_out/):
#   1. the reference arm (the bench line itself comes from a plain `python bench.py` run)
#   2. ncu launch list of the bench command (gpu__time_duration.sum only)
#   3. ncu --set full of the fused pass and of the streamed sketch at the C4 shape
#   4. warm per-kernel profile of a solve (CUPTI)
OUT=gpurun_out
python bench.py > $OUT/rd2f_bench.json 2> $OUT/rd2f_bench.err
[ -n "$SKIP_REF" ] || python bench.py --impl reference --steps 1 --warmup 0 > $OUT/rd2f_bench_ref.json 2> $OUT/rd2f_bench_ref.err
# (ncu cannot profile kernels launched into a green context: the QR's SM partition is switched off for
#  this pass — the results are bitwise the same; the instance generator's library kernels are filtered out)
ITSK_QR_GREEN=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'k_|DeviceRadix|DeviceScan' \
    --log-file $OUT/rd2f_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable > $OUT/rd2f_bench_ncu.log 2>&1
python scripts/pass_ab.py 4000000,2000 > $OUT/rd2f_pass_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_pass_rows -s 3 -c 1 \
    -o $OUT/rd2f_pass_full python scripts/pass_ab.py 4000000,2000 > $OUT/rd2f_pass_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sketch_stream -c 1 \
    -o $OUT/rd2f_sketch_full python scripts/sketch_c4_once.py 4000000 2000 24000 8 1 > $OUT/rd2f_sketch_ncu.log 2>&1
python scripts/kernel_profile.py c4 momentum > $OUT/rd2f_kprof_c4.txt 2>&1
echo done
python bench.py --config c3 --no-cpu-baseline > $OUT/rd2f_bench_c3.json 2> $OUT/rd2f_bench_c3.err
python bench.py --config c2 > $OUT/rd2f_bench_c2.json 2> $OUT/rd2f_bench_c2.err
