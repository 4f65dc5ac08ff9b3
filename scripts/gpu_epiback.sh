#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for eb in 256 64 0; do
  DX_NVCC_EXTRA="-DDX_EPI_BACK=$eb" python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2511_15015_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)"
  for b in 24 60; do
    timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 --no-batch-sweep --no-q80b --budget-gb $b > gpurun_out/sweep.json 2> gpurun_out/sweep.err
    python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read()); r=d['roofline']; x=d['extra']; p=x['prefill']
print('epi_back $eb budget $b: value %.0f gateup %.0f GB/s | prefill %.0f TF/s' % (d['value'], r['achieved'], p['gemm_tflops']))" || tail -3 gpurun_out/sweep.err
  done
done
