run() { timeout 900 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed $2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1 $2', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"; }
for S in 16 32 64; do
USCG_WAVE_PAIR=0 run single "--problems $S"
USCG_WAVE_PAIR=2 run cl2 "--problems $S"
USCG_WAVE_PAIR=4 run cl4 "--problems $S"
done
USCG_WAVE_PAIR=0 run single "--problems 128"
USCG_WAVE_PAIR=2 run cl2 "--problems 128"
