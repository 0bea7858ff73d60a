set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deferred.py -m gpu -q -x -p no:cacheprovider -k "trsv_pair_cluster or solve_parity or deferred or c3_full or estimates" > gpurun_out/g20_pytest.txt 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/g20_pytest.txt | grep -v "^PASSED"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-pageable > gpurun_out/g20_bench_c4.json 2> gpurun_out/g20_bench_c4.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/g20_bench_c4.json; tail -3 gpurun_out/g20_bench_c4.err
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-pageable > gpurun_out/g20_bench_c3.json 2>&1; tail -c 1500 gpurun_out/g20_bench_c3.json
