#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -4 gpurun_out/gpu_tests.log
for b in 16 24 60; do
  echo "== budget $b"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 --budget-gb $b > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read()); r=d['roofline']; x=d['extra']; p=x['prefill']
print('value %.0f gateup %.0f GB/s both %.0f GB/s | prefill %.0f tok/s %.0f TF/s' % (d['value'], r['achieved'], r['ffn_both_phases_gbs'], p['value'], p['gemm_tflops']))" || tail -3 gpurun_out/sweep.err
done
export DX_WATCHDOG_S=120
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 580 -c 2 -o gpurun_out/prof_int4 -f python bench.py --layers 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 --budget-gb 16 > gpurun_out/ncu_int4.log 2>&1
tail -1 gpurun_out/ncu_int4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 624 -c 2 -o gpurun_out/prof_prefill -f python bench.py --layers 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 > gpurun_out/ncu_prefill.log 2>&1
tail -1 gpurun_out/ncu_prefill.log
