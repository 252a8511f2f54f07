run() { timeout 900 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed $2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1 $2', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"; }
for S in 128 64; do
USCG_WAVE_SLOTS=1 run slots1 "--problems $S"
USCG_WAVE_SLOTS=2 run slots2 "--problems $S"
done
