#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read()); r=d['roofline']; x=d['extra']; p=x['prefill']; s=x['switch']
print('value %.0f ms/step %.3f gateup %.0f GB/s frac %.3f | P %d D %d exposed %.4f xfer %.3f ms | prefill %.0f tok/s %.0f TF/s | e2e %.0f' % (d['value'], d['ms_per_step'], r['achieved'], r['frac'], s['promotions'], s['demotions'], s['exposed_frac_of_step_time'], s['xfer_ms_mean'], p['value'], p['gemm_tflops'], d['e2e']['value']))" || tail -3 gpurun_out/bench.err
timeout 600 python bench.py --switch-stress > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "c5 rc=$?"; tail -2 gpurun_out/c5.err
python -c "
import json; d=json.loads(open('gpurun_out/c5.json').read())
for r in d['rows']: print(r['n_hot'], r['mode'], '%.3f ms' % r['ms_per_step'], 'P', r['promotions'], 'D', r['demotions'], 'sw %.3f/%.3f ms' % (r['switch_ms_mean'], r['switch_ms_max']), 'exp %.4f' % r['exposed_frac'])"
bash scripts/gpu_ring.sh 2>&1 | grep -v "^$" | tail -9
