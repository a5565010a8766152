#!/bin/sh
# Fused-rebuild time per phase at a config (RB_REBUILD_STOP=k returns after
# phase k: 7 = binning done, 8 = rows done, 99 = all incl. mirror).
cfg=${1:-cfg4}
for st in 7 8 99; do
  RB_REBUILD_STOP=$st python tools/kernel_bench.py $cfg --skin 0.3 --reps 3 2>/dev/null | \
    python -c "import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('stop', $st, d['config'], 'rebuild_ms', round(d['rebuild_ms'], 4))"
done
