set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
free -g; nproc; lscpu | head -20
./scripts/bw/dmma_peak > gpurun_out/dmma_peak.txt 2>&1
python scripts/bw/dgemm_peak.py > gpurun_out/dgemm_peak.txt 2>&1
cat gpurun_out/dmma_peak.txt gpurun_out/dgemm_peak.txt
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c4_base.json 2> gpurun_out/c4_base.err
tail -c 3000 gpurun_out/c4_base.json; tail -5 gpurun_out/c4_base.err
