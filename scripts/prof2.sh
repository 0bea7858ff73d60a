python -m pytest tests/test_gpu_parity.py -q -x -k "sketch or pattern or digest" 2>&1 | tail -3
for g in 8 4 2; do for u in 2 4 8; do echo "gcpl=$g unr=$u"; ITSK_SKETCH_GCPL=$g ITSK_SKETCH_UNR=$u python scripts/micro_sketch.py 200000 200 4000 8; done; done
for g in 8 4; do for u in 4 8; do echo "gcpl=$g unr=$u"; ITSK_SKETCH_GCPL=$g ITSK_SKETCH_UNR=$u python scripts/micro_sketch.py 4000000 2000 24000 8 2; done; done
for g in 4 2 1; do for u in 4 8; do echo "gcpl=$g unr=$u"; ITSK_SKETCH_GCPL=$g ITSK_SKETCH_UNR=$u python scripts/micro_sketch.py 1048576 100 400 8; done; done
