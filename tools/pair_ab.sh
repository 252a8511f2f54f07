run() { timeout 900 python bench.py --config c2 --steps 20 --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed $2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('PAIR=$1 $2', round(d['ms_per_step'],3), round(d['roofline']['frac'],3))
"; }
for i in 1 2; do USCG_WAVE_PAIR=0 run 0; USCG_WAVE_PAIR=1 run 1; done
USCG_WAVE_PAIR=0 run 0 "--problems 16"; USCG_WAVE_PAIR=1 run 1 "--problems 32"; USCG_WAVE_PAIR=0 run 0 "--problems 32"
