#!/bin/bash
# C2 e2e (uscg_reconstruct_batch) per library build in abtest/
cp paper_2208_12964_b200/lib/libuscg_b200.so /tmp/keep.so
for lib in "$@"; do
  cp abtest/$lib paper_2208_12964_b200/lib/libuscg_b200.so
  timeout 600 python bench.py --config c2 --no-cpu --no-uscg --no-store-fed 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$lib', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'iso', round(d['isolated_iteration']['ms_per_iteration'],3))
"
done
cp /tmp/keep.so paper_2208_12964_b200/lib/libuscg_b200.so
