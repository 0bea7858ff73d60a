#!/bin/bash
# A/B of the sweep's direct mode against the gather / ring / materialised sweep on C5 cells
# (first shape = the previous behaviour and the bitwise reference).  Writes gpurun_out/sketch_direct_ab.txt
OUT=gpurun_out/sketch_direct_ab.txt
: > $OUT
for cell in "16777216 100 400 8" "16777216 100 1200 8" "16777216 100 2000 8" "16777216 100 400 16" \
            "4194304 100 400 8" "4194304 100 2000 16" "4194304 100 1200 4" "1048576 100 400 8" "1048576 100 2000 4" \
            "16777216 500 2000 8" "4194304 500 2000 8" "4194304 500 2000 4" "1048576 500 2000 8" "1048576 500 2000 16"; do
  echo "== $cell" >> $OUT
  timeout 600 python scripts/sketch_sweep_ab.py $cell 3 DIRECT=0,SWCL=0 DIRECT=1,SWCL=0 DIRECT=1,SWCL=2 >> $OUT 2>&1
done
