mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_far_apply|k_far_y" --launch-skip 6 --launch-count 12 -o gpurun_out/qr_far2 -f python scripts/qr_kernels.py 24000 2000 1 > gpurun_out/qr_far_ncu.log 2>&1
tail -3 gpurun_out/qr_far_ncu.log
