run() { timeout 900 python bench.py --config $1 --steps 5 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', 'RUN=${USCG_RUN:-def}', round(d['ms_per_step'],3), d['roofline']['dependency_levels_per_iteration'])
"; }
for r in 1 2 4 8; do USCG_RUN=$r run c4; USCG_RUN=$r run c3; done
