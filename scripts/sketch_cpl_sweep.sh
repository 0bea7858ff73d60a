# gather kernel columns-per-lane at the C4 / C3 shapes (fewer columns per warp -> more resident warps per strip)
for shape in "4000000 2000 24000" "1000000 500 10000"; do
  for g in 1 2 4; do echo -n "GCPL=$g "; ITSK_SKETCH_GCPL=$g python scripts/micro_sketch.py $shape 8 2 | tail -1; done
done
