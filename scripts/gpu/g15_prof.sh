set -x
mkdir -p gpurun_out
python scripts/bw/qrnext2prof.py 24000 2000 > gpurun_out/g15_next2prof.txt 2>&1; cat gpurun_out/g15_next2prof.txt
python scripts/bw/qr2prof.py 24000 2000 > gpurun_out/g15_qr2prof_c4.txt 2>&1; cat gpurun_out/g15_qr2prof_c4.txt
# ncu: one full capture of the C4 pass (the bench's dominant kernel)
timeout 900 ncu --kernel-name regex:k_pass_rows --launch-skip 3 --launch-count 1 --set full --clock-control none \
  --import-source on -o gpurun_out/rd2_pass_c4_full -f python scripts/pass_ab.py 4000000,2000 > gpurun_out/g15_ncu_full.log 2>&1
echo "ncu full rc=$?"
ncu -i gpurun_out/rd2_pass_c4_full.ncu-rep --page raw --csv > gpurun_out/rd2_pass_c4_raw.csv 2>&1
grep -o '"dram__bytes_read.sum[^,]*,[^,]*,[^,]*' gpurun_out/rd2_pass_c4_raw.csv | head; 
# the launch list of the bench command (cold, serialised: shares, not absolutes)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:itsk --csv \
  --log-file gpurun_out/rd2_launches_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-pageable \
  > gpurun_out/g15_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
wc -l gpurun_out/rd2_launches_c4.csv; tail -3 gpurun_out/g15_ncu_launch.log
