#!/bin/bash
# C3 / C4 flow executor A/B: tools/flow_ab.sh "ENV=..." "ENV=..." ...
run() { timeout 900 env $2 python bench.py --config $1 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1 [$2]', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"; }
for c in ${CONFIGS:-c3 c4}; do for e in "$@"; do run $c "$e"; done; done
