#!/bin/bash
# A/B of the length-weighted row action's launch form: tools/lw_ab.sh ["64 128 256"]
# (USCG_CSR_THREADS per line; USCG_CSR_PDL / USCG_CSR_GRAPH off for the last rows)
run() {
  echo -n "threads=$1 pdl=$2 graph=$3: "
  USCG_CSR_THREADS=$1 USCG_CSR_PDL=$2 USCG_CSR_GRAPH=$3 python bench.py --config lw --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(' '.join('%s %.3f ms/it, %d levels (binary %.3f)' % (k, d[k]['ms_per_iteration'], d[k]['levels'], d[k]['binary_model_ms_per_iteration']) for k in ('c1','c3')))"
}
for t in ${1:-64 128 256}; do run $t 1 1; done
run 64 0 1
run 64 1 0
