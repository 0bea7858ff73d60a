# QR kernels under ncu --set full at the C2 and C4 sketch shapes (DMMA pipe utilisation)
set -e
python scripts/micro_qr.py 4000 200 2 > gpurun_out/qr_plain.log
ncu --set full --clock-control none -k regex:"k_qr_(y|apply|next|panel)" -c 8 -o gpurun_out/qr_c2 python scripts/micro_qr.py 4000 200 1 > gpurun_out/qr_c2_ncu.log 2>&1
ncu --set full --clock-control none -k regex:"k_qr_(y|apply|panel)" -s 12 -c 6 -o gpurun_out/qr_c4 python scripts/micro_qr.py 24000 2000 1 > gpurun_out/qr_c4_ncu.log 2>&1
echo done
