set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "fused_pass or solve_parity" > gpurun_out/g4_pytest.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/g4_pytest.txt
for v in 0 1; do ITSK_PASS_ROWCTA=$v timeout 300 python scripts/pass_ab.py 2000000,1000 1000000,600 1000000,513 2000000,800 4000000,2000 ; done > gpurun_out/g4_pass_ab.txt 2>&1
cat gpurun_out/g4_pass_ab.txt
timeout 600 python scripts/kernel_profile.py c4 momentum > gpurun_out/g4_kprof_c4.txt 2>&1
cat gpurun_out/g4_kprof_c4.txt
