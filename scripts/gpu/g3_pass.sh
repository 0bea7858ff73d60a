set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "fused_pass or solve_parity or c2_shape" > gpurun_out/g3_pytest.txt 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/g3_pytest.txt
ITSK_PASS_ROWCTA=0 timeout 300 python scripts/pass_ab.py 4000000,2000 1000000,2000 2000000,1000 500000,1536 > gpurun_out/g3_pass_old.txt 2>&1
ITSK_PASS_ROWCTA=1 timeout 300 python scripts/pass_ab.py 4000000,2000 1000000,2000 2000000,1000 500000,1536 > gpurun_out/g3_pass_new.txt 2>&1
cat gpurun_out/g3_pass_old.txt gpurun_out/g3_pass_new.txt
