python -m pytest tests/test_gpu_parity.py -q -x -k "sketch or pattern or digest" 2>&1 | tail -2
python scripts/micro_sketch.py 200000 200 4000 8
python scripts/micro_sketch.py 1000000 500 10000 8
python scripts/micro_sketch.py 1048576 100 400 8
python scripts/micro_sketch.py 1048576 2000 8000 4 2
python scripts/bw/qrprof.py 24000 2000
python scripts/bw/qrprof.py 10000 500
python scripts/bw/qrprof.py 4000 200
python scripts/micro_qr.py 24000 2000 2>&1 | tail -3
ITSK_QR_MODE=tsqr python scripts/micro_qr.py 24000 2000 2>&1 | tail -3
