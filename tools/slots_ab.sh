run() { timeout 900 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu --no-uscg --no-store-fed 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('SLOTS=${USCG_BATCH_SLOTS:-2}', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3))
"; }
for n in 2 3 4 2 3; do USCG_BATCH_SLOTS=$n run; done
