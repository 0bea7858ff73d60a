mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:k_sketch_sweep --launch-count 1 -o gpurun_out/sk_sweep3 -f python scripts/sketch_c4_once.py 4000000 2000 24000 8 1 > gpurun_out/sk_sweep3_ncu.log 2>&1
tail -5 gpurun_out/sk_sweep3_ncu.log
