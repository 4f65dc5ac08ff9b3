#!/bin/bash
# exposed switch time attribution: C2 bench switch leg and C5 with the demotions' quantisation (DX_XFER_SKIP=1) or the
# promotions' copies (DX_XFER_SKIP=2) skipped (timing only: the moved experts' weights are then wrong)
python __graft_entry__.py > /dev/null 2>&1 || exit 1
for sk in 0 1 2; do
  DX_XFER_SKIP=$sk timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-prefetch-leg --no-q80b --no-batch-sweep --prefill-tokens 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]);s=d['extra']['switch']
print('C2 DX_XFER_SKIP=$sk on',round(s['on_ms_per_step'],3),'tele',round(s['teleport_ms_per_step'],3),'exposed',round(s['exposed_frac_teleport'],4))"
  DX_XFER_SKIP=$sk timeout 900 python bench.py --switch-stress 2>/dev/null | python -c "
import json,sys
c=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('C5 DX_XFER_SKIP=$sk', [(r['n_hot'], r['mode'][0], round(r['exposed_frac_teleport'],3)) for r in c['rows'] if r['n_hot'] in (13, 64, 115)])"
done
