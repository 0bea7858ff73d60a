set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "sketch or pattern or chunked or c3_full" > gpurun_out/g18_pytest.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g18_pytest.txt
python scripts/sketch_c4_once.py 4000000 2000 24000 8 3
ITSK_SKETCH_WIN=0 python scripts/sketch_c4_once.py 4000000 2000 24000 8 2
python scripts/sketch_c4_once.py 1000000 500 10000 8 3
ITSK_SKETCH_WIN=0 python scripts/sketch_c4_once.py 1000000 500 10000 8 2
python scripts/sketch_c4_once.py 200000 200 4000 8 3
python scripts/pass_ab.py 1000000,500 1000000,500 200000,200
