# usage (gpurun): bash tools/ab.sh c2 c3 ...   (build abtest/libA.so first: bash tools/ab_mklib.sh)
# A/B: abtest/libA.so versus the working tree's library, same box; args: configs...
set -e
rm -rf /tmp/A && cp -r "$GRAFT_REPO_ROOT" /tmp/A && cp abtest/libA.so /tmp/A/paper_2208_12964_b200/lib/libuscg_b200.so && touch /tmp/A/paper_2208_12964_b200/lib/libuscg_b200.so
run() { timeout 900 python bench.py --config $2 --steps ${STEPS:-20} --warmup 2 --no-cpu --no-e2e --no-uscg --no-store-fed 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', '$2', round(d['ms_per_step'],3))
"; }
for cfg in "$@"; do
  for i in 1 2; do
    (cd /tmp/A && run A $cfg)
    run B $cfg
  done
done
