# C2-shape fused-pass knob sweep (tile bytes, ring budget, CTAs per SM)
for cps in 1 2; do for tb in 8192 16384 32768; do for sk in 96 200; do
  echo -n "ctas/sm=$cps tile=$tb smem=${sk}KB: "
  ITSK_PASS_CTAS_PER_SM=$cps ITSK_PASS_TILE_BYTES=$tb ITSK_PASS_SMEM_KB=$sk python scripts/micro_pass.py 200000 200 50
done; done; done
python scripts/micro_pass.py 1000000 500 20
python scripts/micro_pass.py 400000 200 20
python scripts/micro_pass.py 800000 200 20
