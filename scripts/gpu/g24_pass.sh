set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_deferred.py tests/test_gpu_dist.py tests/test_gpu_lsqr.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python scripts/pass_ab.py 200000,200 800000,200 1000000,300 4000,50 1000000,100 4000000,2000
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-pageable > gpurun_out/g24_bench_c2.json 2>&1; tail -c 2500 gpurun_out/g24_bench_c2.json
