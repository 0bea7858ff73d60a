set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "qr or solve_parity or c2_shape or trsv or estimates or condest" > gpurun_out/g11_pytest.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g11_pytest.txt
python scripts/micro_qr.py 24000 2000 5; python scripts/micro_qr.py 4000 200 20; python scripts/micro_qr.py 10000 500 10
python scripts/qr_kernels.py 24000 2000 > gpurun_out/g11_qrk_c4.txt 2>&1; cat gpurun_out/g11_qrk_c4.txt
python scripts/qr_kernels.py 10000 500 > gpurun_out/g11_qrk_c3.txt 2>&1; cat gpurun_out/g11_qrk_c3.txt
