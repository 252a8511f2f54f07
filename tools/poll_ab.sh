#!/bin/bash
# C2 wave executor: poller back-off / publisher sleep, and pairs at 128 problems
run() { timeout 900 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"; }
USCG_WAVE_PAIR=0 run "default"
for pn in 64 128 512; do USCG_WAVE_PAIR=0 USCG_WAVE_POLL_NS=$pn run "poll_ns=$pn"; done
for pb in 0 16 64 128; do USCG_WAVE_PAIR=0 USCG_WAVE_PUB_NS=$pb run "pub_ns=$pb"; done
USCG_WAVE_PAIR=2 run "pairs at 128"
USCG_WAVE_PAIR=0 run "default"
