#!/bin/bash
# A/B of the sweep's direct mode (DIRECT=1) and the gated ring (DIRECT=2) against the previous choice
# (DIRECT=0: ring / gather / materialised sweep; the bitwise reference) on C5 cells.  Writes gpurun_out/sketch_direct_ab.txt
OUT=gpurun_out/sketch_direct_ab.txt
: > $OUT
for cell in "16777216 100 400 8" "16777216 100 1200 8" "16777216 100 2000 8" "16777216 100 400 16" \
            "4194304 100 400 8" "4194304 100 2000 16" "4194304 100 1200 4" "1048576 100 400 8" "1048576 100 2000 4" \
            "1048576 100 1200 16" "16777216 500 2000 8" "4194304 500 2000 8" "4194304 500 2000 4" "1048576 500 2000 8"; do
  echo "== $cell" >> $OUT
  timeout 600 python scripts/sketch_sweep_ab.py $cell 3 DIRECT=0,SWCL=0 ${SHAPES:-DIRECT=1 DIRECT=2} >> $OUT 2>&1
done
