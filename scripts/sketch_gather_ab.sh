OUT=gpurun_out/sketch_gather_ab.txt
: > $OUT
for cell in "16777216 100 1200 8" "16777216 100 2000 8" "4194304 100 2000 16" "4194304 100 1200 4" "16777216 100 400 8"; do
  echo "== $cell" >> $OUT
  timeout 600 python scripts/sketch_sweep_ab.py $cell 3 DIRECT=0,SWCL=0 GCPL=1,UNR=8 GCPL=2,UNR=8 GCPL=2,UNR=4 GCPL=4,UNR=4 GCPL=4,UNR=8 >> $OUT 2>&1
done
