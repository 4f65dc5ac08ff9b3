#!/bin/bash
# side-stream transition block count: default bench value (plan period inside the timed region) and C5 exposure
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for nb in 148 32 8; do
  DX_NVCC_EXTRA="-DDX_XFER_BLOCKS=$nb" python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_2511_15015_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)"
  echo "#### xfer blocks $nb"
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --prefill-tokens 0 > gpurun_out/bench.json 2> gpurun_out/bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read()); r=d['roofline']; x=d['extra']; s=x['switch']
print('value %.0f ms/step %.3f gateup %.0f GB/s | P %d D %d exposed %.4f xfer %.3f ms | e2e %.0f' % (d['value'], d['ms_per_step'], r['achieved'], s['promotions'], s['demotions'], s['exposed_frac_of_step_time'], s['xfer_ms_mean'], d['e2e']['value']))" || tail -3 gpurun_out/bench.err
  timeout 600 python bench.py --switch-stress > gpurun_out/c5_$nb.json 2> gpurun_out/c5.err
  python -c "
import json; d=json.loads(open('gpurun_out/c5_$nb.json').read())
print('C5 max exposed %.4f' % d['value'], ' decode sw ms', ['%.2f' % r['switch_ms_mean'] for r in d['rows'] if r['mode']=='decode'][:3], ' decode ms/step', ['%.3f' % r['ms_per_step'] for r in d['rows'] if r['mode']=='decode'][:3])"
done
