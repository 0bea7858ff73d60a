#!/bin/bash
# old-vs-new A/B of the register gather in one GPU call (libitsk_b200_old.so = the previous sketch.cu)
cd paper_2311_04362_b200; cp libitsk_b200.so /tmp/new.so; cp libitsk_b200_old.so /tmp/old.so; cd ..
: > gpurun_out/s5_gather_oldnew.txt
for rep in 1 2; do
for v in new old; do
  cp /tmp/$v.so paper_2311_04362_b200/libitsk_b200.so
  echo "== $v" >> gpurun_out/s5_gather_oldnew.txt
  for cell in "200000 200 4000 8" "16777216 100 2000 8" "4194304 100 1200 16" "4194304 500 2000 8" "1048576 500 6000 8" "1048576 500 10000 4" "4000000 2000 24000 8"; do
    python scripts/sketch_c4_once.py $cell 4 2>&1 | tail -1 >> gpurun_out/s5_gather_oldnew.txt
  done
done; done
cp /tmp/new.so paper_2311_04362_b200/libitsk_b200.so
