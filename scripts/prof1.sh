set -x
mkdir -p gpurun_out
python scripts/micro_pass.py 4000000 2000 10
python scripts/micro_pass.py 200000 200 50
python scripts/micro_pass.py 1000000 500 30
python scripts/micro_sketch.py 200000 200 4000 8
python scripts/micro_sketch.py 1000000 500 10000 8
python scripts/micro_sketch.py 4000000 2000 24000 8 2
python scripts/micro_sketch.py 1048576 100 400 8
python scripts/micro_sketch.py 16777216 100 2000 16 2
ncu --set full --clock-control none --import-source on -k regex:k_sketch_gather -c 1 -o gpurun_out/sketch_c2 -f python scripts/micro_sketch.py 200000 200 4000 8 1 > gpurun_out/ncu_sketch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass -c 1 -o gpurun_out/pass_c4 -f python scripts/micro_pass.py 4000000 2000 1 > gpurun_out/ncu_pass.log 2>&1
ls -la gpurun_out
