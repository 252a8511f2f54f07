#!/bin/bash
# A/B of library builds in abtest/: tools/lib_ab.sh "<bench args>" libA.so libB.so ...
args=$1; shift
cp paper_2208_12964_b200/lib/libuscg_b200.so /tmp/lib_keep.so
for lib in "$@"; do
  cp abtest/$lib paper_2208_12964_b200/lib/libuscg_b200.so
  timeout 900 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed $args 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$lib $args', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"
done
cp /tmp/lib_keep.so paper_2208_12964_b200/lib/libuscg_b200.so
