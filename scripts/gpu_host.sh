#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for pdl in 1 0; do
DX_PDL=$pdl timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --prefill-tokens 0 --no-batch-sweep --no-q80b > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read())
print('PDL=$pdl value %.0f ms/step %.3f host_issue_ms/step %.3f e2e %.0f' % (d['value'], d['ms_per_step'], d['extra']['host_issue_ms_per_step'], d['e2e']['value']))" || tail -3 gpurun_out/bench.err
done
