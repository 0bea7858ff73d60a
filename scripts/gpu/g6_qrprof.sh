set -x
mkdir -p gpurun_out
python scripts/bw/qr2prof.py 24000 2000 > gpurun_out/g6_qr2prof_c4.txt 2>&1
python scripts/bw/qr2prof.py 4000 200 > gpurun_out/g6_qr2prof_c2.txt 2>&1
python scripts/bw/qr2prof.py 10000 500 > gpurun_out/g6_qr2prof_c3.txt 2>&1
cat gpurun_out/g6_qr2prof_*.txt
python scripts/micro_qr.py 24000 2000 5; python scripts/micro_qr.py 4000 200 20; python scripts/micro_qr.py 10000 500 10
