set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "fused_pass" > gpurun_out/g17_pytest.txt 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/g17_pytest.txt
python scripts/pass_ab.py 4000000,2000 1000000,500
python scripts/sketch_c4_once.py 4000000 2000 24000 8 3
timeout 600 ncu --kernel-name regex:k_sketch_gather --launch-count 1 --section SpeedOfLight --section MemoryWorkloadAnalysis --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct --clock-control none python scripts/sketch_c4_once.py 4000000 2000 24000 8 1 > gpurun_out/g17_sketch_ncu.txt 2>&1
grep -E "dram__bytes|lts__t_sector|Duration|Throughput|Hit" gpurun_out/g17_sketch_ncu.txt | head -30
