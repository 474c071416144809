for g in 148 96 74 48 37; do DS_PCG_GRID=$g timeout 200 python scripts/r02/pcg_time.py 0 20 2>&1 | tail -1 | sed "s/^/grid $g: /"; done
