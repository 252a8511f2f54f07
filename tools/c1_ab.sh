#!/bin/bash
cp paper_2208_12964_b200/lib/libuscg_b200.so /tmp/keep.so
for lib in "$@"; do
  cp abtest/$lib paper_2208_12964_b200/lib/libuscg_b200.so
  timeout 600 python bench.py --config c1 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$lib c1', round(d['ms_per_step'],4))
"
done
cp /tmp/keep.so paper_2208_12964_b200/lib/libuscg_b200.so
