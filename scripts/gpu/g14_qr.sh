set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "qr or c2_shape" > gpurun_out/g14_pytest.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g14_pytest.txt
python scripts/micro_qr.py 24000 2000 5; python scripts/micro_qr.py 16500 1100 5
python scripts/qr_kernels.py 24000 2000 > gpurun_out/g14_qrk_c4.txt 2>&1; cat gpurun_out/g14_qrk_c4.txt
