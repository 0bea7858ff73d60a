set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_guards.py -m gpu -q -x -p no:cacheprovider -rA > gpurun_out/g19_guards.txt 2>&1; echo "guards rc=$?"
tail -25 gpurun_out/g19_guards.txt | grep -v "^PASSED"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/g19_pytest.txt 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/g19_pytest.txt
