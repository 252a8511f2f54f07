#!/bin/bash
# clustered wave: poller back-off per stack size (chain-bound small stacks)
for S in ${SIZES:-16 32 128}; do
  for pn in 256 64 16; do
    echo "S=$S poll_ns=$pn $(USCG_WAVE_POLL_NS=$pn timeout 600 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed --problems $S 2>/dev/null | python -c "import json,sys; [print(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin if l.startswith('{')]")"
  done
done
