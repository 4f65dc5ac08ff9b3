#!/bin/bash
# k_wide check: prefill-path GPU tests, then the C3 prefill leg with and without k_wide (DX_WIDE=0).
mkdir -p gpurun_out
TAG=${1:-wide}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
DX_WATCHDOG_S=20 timeout 1200 python -m pytest tests -m gpu -x -q -k "${TESTK:-4096 or prefill or paper_shape or shared or route}" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
for w in 1 0; do
  DX_WIDE=$w DX_WATCHDOG_S=20 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-batch-sweep --no-teleport --no-prefetch-leg > gpurun_out/${TAG}_bench_w$w.json 2> gpurun_out/${TAG}_bench_w$w.err; echo "bench DX_WIDE=$w rc=$?"
  python - gpurun_out/${TAG}_bench_w$w.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
p=d['extra']['prefill']; q=d['extra'].get('q80b',{}).get('prefill',{})
print(f"  decode {d['value']:.0f} ms/step {d['ms_per_step']:.3f} | prefill {p['value']:.0f} tok/s ms/step {p['ms_per_step']:.2f} gemm {p['gemm_tflops']:.0f} TF/s frac {p['tensor_frac']:.3f} share {p['gemm_ms_share']:.3f} | q80b prefill {q.get('gemm_tflops',0):.0f} TF/s")
PY
done
