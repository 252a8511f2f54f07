#!/bin/bash
# updater warps per SM of the list-fed dataflow executor: tools/groups_ab.sh c4 "20 24 28 32"
cfg=${1:-c4}
for g in ${2:-"20 32"}; do
  echo -n "$cfg groups=$g: "
  USCG_FLOW_VERBOSE=1 USCG_UPD_GROUPS=$g python bench.py --config $cfg 2>gpurun_out/groups_$g.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('ms/it', round(d['ms_per_iteration'],3), 'e2e', round(d['e2e']['ms_per_step'],3))"
  grep -m1 "mart_flow_kernel:" gpurun_out/groups_$g.err
done
