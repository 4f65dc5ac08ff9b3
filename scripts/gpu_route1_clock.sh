#!/bin/bash
# phase clocks of k_route1 (debug build with -DDX_ROUTE_PROF; printed once, at the 300th call)
mkdir -p gpurun_out
DX_NVCC_EXTRA="-DDX_ROUTE_PROF" python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2511_15015_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)"
timeout 300 python bench.py --layers 8 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep 2>&1 | grep route1
