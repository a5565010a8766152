#!/bin/sh
# Fused-rebuild phase times (rows, rows + mirror) and the separate rows +
# mirror launch time for a list of library builds (RB_LIB_PATH; "base" = the
# in-tree library):  sh tools/rebuild_ab.sh cfg4 base build/lib_x.so ...
cfg=$1; shift
for lib in "$@"; do
  L=$lib; [ "$lib" = base ] && L=""
  for st in 8 99; do
    RB_LIB_PATH=$L RB_REBUILD_STOP=$st python tools/kernel_bench.py $cfg --skin 0.3 --reps 5 2>/dev/null | \
      python -c "import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$lib', 'stop', $st, d['config'], 'rebuild_ms', round(d['rebuild_ms'], 4), 'nlist_ms', round(d['nlist_ms'], 4))"
  done
done
