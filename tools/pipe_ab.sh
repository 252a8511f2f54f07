#!/bin/bash
# clustered wave form: plain vs pipelined (USCG_WAVE_PIPE) per C2 stack size
run() { timeout 900 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed $2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1 $2', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"; }
for S in ${SIZES:-16 32 64 128}; do
USCG_WAVE_PIPE=0 run plain "--problems $S"
USCG_WAVE_PIPE=1 run pipe "--problems $S"
done
