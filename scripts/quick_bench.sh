#!/bin/bash
# quick_bench.sh TAG WORKLOAD... : one short bench line per workload, condensed (GPU box helper)
tag=$1; shift
for w in "$@"; do
  python bench.py --workload $w --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline']
print('$tag', d['config']['workload'], round(d['value']), d['ms_per_step'], {k:round(v*1e3,1) for k,v in r.get('slot_ms_per_step',{}).items()})"
done
