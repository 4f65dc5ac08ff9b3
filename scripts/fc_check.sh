#!/bin/bash
# fused combine check: GPU tests, one-layer timings, C2 bench (switch leg) at two demotion grid sizes
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
DX_WATCHDOG_S=20 timeout 1500 python -m pytest tests -m gpu -x -q ${TESTK:+-k "$TESTK"} > gpurun_out/fc_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fc_tests.log
for cfg in "24 1 1.2" "24 16 1.2" "24 64 1.2" "0 64 1.2"; do DX_WATCHDOG_S=10 QD_ROUTER=1 timeout 120 python scripts/qd_one.py $cfg 256 2>&1 | tail -1; done
for db in ${DBS:-148 16}; do
  DX_DEMOTE_BLOCKS=$db timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-prefetch-leg --no-q80b --no-batch-sweep --prefill-tokens 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d['roofline'];x=d['extra']
print('DX_DEMOTE_BLOCKS=$db value',round(d['value']),'ms',round(d['ms_per_step'],3),'frac',round(r['frac'],3),'layer',round(r['layer_frac'],3),'exposed',round(x['switch']['exposed_frac_teleport'],4),'tele',round(x['switch']['teleport_ms_per_step'],3),'launches',d['gpu_launches'])"
done
