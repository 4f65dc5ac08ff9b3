#!/bin/bash
# one GPU iteration: build, gpu tests, default bench, tier sweep; "ncu" adds a --set full capture of the
# steady-state (mixed-tier) decode GEMMs (8-layer stack: skip the controller warm-up's 32*8*2 launches)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -4 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
for cfg in "--budget-gb 60" "--budget-gb 16"; do
  echo "== $cfg"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 $cfg > gpurun_out/sweep.json 2> gpurun_out/sweep.err
  python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read()); r=d['roofline']; x=d['extra']
print('value %.0f ms/step %.2f gateup %.0f GB/s both %.0f GB/s bytes/layer %.1f MB ffn_share %.2f' % (d['value'], d['ms_per_step'], r['achieved'], r['ffn_both_phases_gbs'], x['weight_bytes_per_layer']/1e6, x['ffn_ms_share']))" || tail -5 gpurun_out/sweep.err
done
if [ "$1" == "ncu" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm' -s 580 -c 2 -o gpurun_out/prof_gemm_mixed -f python bench.py --layers 8 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
fi
