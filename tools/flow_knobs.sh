#!/bin/bash
# C3/C4 flow executor variants (library builds in abtest/)
run() { timeout 600 env $3 python bench.py --config $2 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1 $2 [$3]', round(d['ms_per_step'],3))
"; }
cp paper_2208_12964_b200/lib/libuscg_b200.so /tmp/keep.so
for c in ${CONFIGS:-c3 c4}; do
for lib in ${LIBS:-libBase.so libCta1024.so}; do
  cp abtest/$lib paper_2208_12964_b200/lib/libuscg_b200.so
  run $lib $c USCG_FLOW_VERBOSE=0
done
done
cp /tmp/keep.so paper_2208_12964_b200/lib/libuscg_b200.so
