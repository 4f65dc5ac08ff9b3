#!/bin/bash
# A/B of in-tree libdx build variants (DX_LIB=...) on the C2 decode stack: bash scripts/ab_libs.sh "libA.so libB.so" "budget1 budget2"
run() {
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; x=d['extra']
print('value %.0f ms/step %.3f gateup %.0f GB/s (%.3f) both %.0f GB/s (%.3f)' % (d['value'], d['ms_per_step'], r['achieved'], r['frac'], r['ffn_both_phases_gbs'], r['ffn_both_frac']))"
}
for lib in $1; do for b in ${2:-16 24}; do echo "$lib budget $b: $(DX_LIB=$lib run --budget-gb $b)"; done; done
