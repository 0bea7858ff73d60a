for tb in 16384 32768 65536; do for sk in 200 220; do echo "tile=$tb smem=$sk"; ITSK_PASS_TILE_BYTES=$tb ITSK_PASS_SMEM_KB=$sk python scripts/micro_pass.py 1000000 2000 10; done; done
python scripts/micro_pass.py 1000000 1000 10
python scripts/micro_pass.py 1000000 500 10
python scripts/micro_pass.py 2000000 256 10
python scripts/micro_pass.py 4000000 128 10
