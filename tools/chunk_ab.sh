#!/bin/bash
# C2 (128 problems) per-iteration time by chunk width and CTA form
run() { timeout 900 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"; }
for cw in 32 16 8; do
  for pair in 0 2; do
    USCG_FLOW_VERBOSE=1 USCG_CHUNK_WIDTH=$cw USCG_WAVE_PAIR=$pair run "chunk=$cw pair=$pair" 2> >(grep mart_wave >&2)
  done
done
