timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "sketch or c3_full" 2>&1 | tail -2
python scripts/sketch_c4_once.py 4000000 2000 24000 8 4
python bench.py --steps 10 --warmup 3 --no-pageable 2>&1 | tail -1 > gpurun_out/bench_c4_sweep.json
cat gpurun_out/bench_c4_sweep.json | head -c 1500
