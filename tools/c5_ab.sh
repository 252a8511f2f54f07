#!/bin/bash
# A/B of library builds in abtest/ on the C5 generator: tools/c5_ab.sh libA.so libB.so ...
cp paper_2208_12964_b200/lib/libuscg_b200.so /tmp/lib_keep.so
for rep in 1 2; do
for lib in "$@"; do
  cp abtest/$lib paper_2208_12964_b200/lib/libuscg_b200.so
  timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$lib', round(d['generator']['ms'],2), 'rotated', round(d['rotated_reuse']['ms'],1), 'resample', round(d['resample']['ms'],3))
"
done
done
cp /tmp/lib_keep.so paper_2208_12964_b200/lib/libuscg_b200.so
