#!/bin/bash
# old-vs-new A/B of the sketch in one GPU call: paper_2311_04362_b200/libitsk_b200_old.so is a build with the
# previous sketch.cu; both libraries alternate over the same shapes.  CELLS overrides the shapes.
cd paper_2311_04362_b200; cp libitsk_b200.so /tmp/new.so; cp libitsk_b200_old.so /tmp/old.so; cd ..
: > gpurun_out/s5_sketch_oldnew.txt
for rep in 1 2 3; do
for v in new old; do
  cp /tmp/$v.so paper_2311_04362_b200/libitsk_b200.so
  echo "== $v" >> gpurun_out/s5_sketch_oldnew.txt
  python scripts/sketch_c4_once.py 4000000 2000 24000 8 5 2>&1 | tail -2 >> gpurun_out/s5_sketch_oldnew.txt
  python scripts/sketch_c4_once.py 1000000 500 10000 8 5 2>&1 | tail -1 >> gpurun_out/s5_sketch_oldnew.txt
done; done
cp /tmp/new.so paper_2311_04362_b200/libitsk_b200.so
