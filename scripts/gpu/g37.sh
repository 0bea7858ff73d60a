python scripts/phases.py c4 momentum 2>&1 | tail -22
python scripts/loop_timeline.py c2 basic 2>&1 | tail -25
