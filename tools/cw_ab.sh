#!/bin/bash
# C2 per-GPU stack sizes: chunk width 32 vs 16 (pairs)
run() { timeout 600 env $3 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed --problems $2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1 S=$2', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"; }
for S in 16 32 48 64 96 128; do
  run cw32 $S USCG_CHUNK_WIDTH=32
  run cw16 $S USCG_CHUNK_WIDTH=16
done
