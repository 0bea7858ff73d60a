python scripts/solve_ab.py c4 momentum ITSK_SKETCH_SWEEP= ITSK_SKETCH_SWEEP=0 5
