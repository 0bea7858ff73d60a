cd paper_2311_04362_b200; cp libitsk_b200.so /tmp/new.so; cp libitsk_b200_old.so /tmp/old.so; cd ..
: > gpurun_out/s5_ring_oldnew.txt
for rep in 1 2; do
for v in new old; do
  cp /tmp/$v.so paper_2311_04362_b200/libitsk_b200.so
  echo "== $v" >> gpurun_out/s5_ring_oldnew.txt
  python scripts/sketch_c4_once.py 16777216 100 400 8 3 >> gpurun_out/s5_ring_oldnew.txt 2>&1
  python scripts/sketch_c4_once.py 4194304 100 400 16 3 >> gpurun_out/s5_ring_oldnew.txt 2>&1
  python scripts/sketch_c4_once.py 1048576 100 400 4 3 >> gpurun_out/s5_ring_oldnew.txt 2>&1
done; done
cp /tmp/new.so paper_2311_04362_b200/libitsk_b200.so
