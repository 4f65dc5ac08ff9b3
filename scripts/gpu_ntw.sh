#!/bin/bash
# tests at the default transform-warp count, then the decode bench + tier sweep for NTW = 16 and 8
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -4 gpurun_out/gpu_tests.log
for ntw in 16 8; do
  echo "#### NTW=$ntw"
  DX_NVCC_EXTRA="-DDX_GEMM_NTW=$ntw" python -c "import sys; sys.path.insert(0,'.'); import importlib.util as u; s=u.spec_from_file_location('b','paper_2511_15015_b200/build.py'); b=u.module_from_spec(s); s.loader.exec_module(b); b.build(force=True)"
  for cfg in "--budget-gb 24" "--budget-gb 60" "--budget-gb 16"; do
    echo "== $cfg"
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 4096 --prefill-steps 2 $cfg > gpurun_out/sweep.json 2> gpurun_out/sweep.err
    python -c "
import json; d=json.loads(open('gpurun_out/sweep.json').read()); r=d['roofline']; x=d['extra']; p=x['prefill']
print('value %.0f ms/step %.2f gateup %.0f GB/s both %.0f GB/s bytes/layer %.1f MB ffn_share %.2f | prefill %.0f tok/s %.0f TF/s' % (d['value'], d['ms_per_step'], r['achieved'], r['ffn_both_phases_gbs'], x['weight_bytes_per_layer']/1e6, x['ffn_ms_share'], p['value'], p['gemm_tflops']))" || tail -5 gpurun_out/sweep.err
  done
done
