#!/bin/bash
# one-layer decode timing (scripts/qd_one.py) across the in-tree libdx variants given as arguments
mkdir -p gpurun_out
for v in "$@"; do
  IFS=, read -ra CL <<< "${CFGS:-0 64 1.2,24 64 1.2,128 64 1.2}"
  for cfg in "${CL[@]}"; do
    echo -n "$v: "; DX_LIB=$([ "$v" = base ] && echo libdx.so || echo libdx_$v.so) DX_WATCHDOG_S=10 timeout 120 python scripts/qd_one.py $cfg 2>&1 | tail -1
  done
done
