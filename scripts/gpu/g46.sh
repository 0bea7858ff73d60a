timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -x -p no:cacheprovider -k "qr" 2>&1 | tail -2
python scripts/qr_kernels.py 24000 2000 3 2>&1 | grep -v Warn | grep "wall\|k_far_t"
python scripts/qr_timeline.py 24000 2000 2>&1 | grep -v arn | grep -A6 "gap totals by the kernel"
