set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -x -p no:cacheprovider -k "fused_pass" 2>&1 | tail -2
for v in 0 1; do ITSK_DEV_PASS_ROWS=$v python scripts/pass_ab.py 4000000,2000 2000000,1000 1000000,500; done
ITSK_DEV_PASS_ROWS=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -x -p no:cacheprovider -k "fused_pass" 2>&1 | tail -2
