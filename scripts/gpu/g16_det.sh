set -x
python scripts/determinism_check.py 24000 2000 4000000
ITSK_QR_LOOKAHEAD=0 python scripts/determinism_check.py 24000 2000
python scripts/determinism_check.py 10000 500
ITSK_QR_LOOKAHEAD=0 python scripts/determinism_check.py 10000 500
./scripts/bw/l2_gather
