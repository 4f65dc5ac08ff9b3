#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for tb in 0 32 100; do
  DX_NVCC_EXTRA="-DDX_TBACK=$tb" python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2511_15015_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)"
  for b in 16 24; do
    echo "== tback $tb budget $b"
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 --no-batch-sweep --budget-gb $b > gpurun_out/sweep.json 2> gpurun_out/sweep.err
    python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read()); r=d['roofline']; x=d['extra']; p=x['prefill']
print('value %.0f gateup %.0f GB/s both %.0f GB/s | prefill %.0f tok/s %.0f TF/s' % (d['value'], r['achieved'], r['ffn_both_phases_gbs'], p['value'], p['gemm_tflops']))" || tail -3 gpurun_out/sweep.err
  done
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --prefill-tokens 0 --no-batch-sweep > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read()); print('value %.0f clocks %s' % (d['value'], d.get('clocks')))" || tail -3 gpurun_out/bench.err
