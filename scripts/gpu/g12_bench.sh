set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "qr" > gpurun_out/g12_pytest.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g12_pytest.txt
python scripts/micro_qr.py 24000 2000 5
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/g12_bench_c4.json 2> gpurun_out/g12_bench_c4.err
echo "bench rc=$?"
tail -c 4000 gpurun_out/g12_bench_c4.json; tail -5 gpurun_out/g12_bench_c4.err
