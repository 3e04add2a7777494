#!/bin/bash
# A/B of library builds on one box: tools/ab.sh "<bench args>" lib1.so lib2.so ...
# prints value / ms per step / depth-1 field launch ms per library (alternating twice)
ARGS=$1; shift
for rep in 1 2; do
  for L in "$@"; do
    WFPG_LIB=$L python bench.py $ARGS --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
r=d['roofline']
print('$L', '%.1f M/s' % (d['value']/1e6), '%.3f ms/step' % d['ms_per_step'], 'd1 %.3f ms' % r['launch_ms'], 'fields %.2f' % r['field_share_of_step'])
"
  done
done
