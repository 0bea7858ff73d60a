# round-2 call 2: full GPU suite with the new tests, the strict-bar table
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rA --durations=25 > gpurun_out/g2_pytest.txt 2>&1
echo "pytest rc=$?"
tail -60 gpurun_out/g2_pytest.txt
timeout 600 python scripts/strict_bar.py > gpurun_out/g2_strict_bar.txt 2>&1
cat gpurun_out/g2_strict_bar.txt
