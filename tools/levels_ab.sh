#!/bin/bash
# the level executor's launch form on C3: tools/levels_ab.sh
run() {
  echo -n "threads=$1 pdl=$2 graph=$3: "
  USCG_MART_MODE=levels USCG_LEVEL_THREADS=$1 USCG_LEVEL_PDL=$2 USCG_LEVEL_GRAPH=$3 python bench.py --config c3 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%.3f ms/it, e2e %.3f, isolated %.3f' % (d['ms_per_iteration'], d['e2e']['ms_per_step'], d['isolated_iteration']['ms_per_iteration']))"
}
run 512 1 0
run 512 1 1
run 256 1 0
