#!/bin/bash
# fused decode FFN check: GPU tests, then one-layer decode timings with and without it (DX_FUSE=0)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
DX_WATCHDOG_S=20 timeout 1500 python -m pytest tests -m gpu -x -q ${TESTK:+-k "$TESTK"} > gpurun_out/fuse_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fuse_tests.log
for f in 1 0; do for cfg in "24 1 1.2" "24 16 1.2" "24 64 1.2" "0 64 1.2" "128 64 1.2"; do echo -n "DX_FUSE=$f "; DX_FUSE=$f DX_WATCHDOG_S=10 QD_ROUTER=1 timeout 120 python scripts/qd_one.py $cfg 256 2>&1 | tail -1; done; done
