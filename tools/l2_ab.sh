#!/bin/bash
# C2 wave executor: L2 eviction priorities of field rows and traced lists (USCG_WAVE_L2)
run() { timeout 900 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"; }
for h in ${@:-00 21 01 20 00}; do USCG_WAVE_PAIR=0 USCG_WAVE_L2=$h run "l2=$h"; done
