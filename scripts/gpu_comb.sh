#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ep.py -x -q --timeout 600 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --prefill-tokens 0 --no-batch-sweep --no-q80b > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read())
print('value %.0f ms/step %.3f e2e %.0f' % (d['value'], d['ms_per_step'], d['e2e']['value']))" || tail -3 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_combine' -s 2000 -c 50 --csv --log-file gpurun_out/launches_comb.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --prefill-tokens 0 --no-batch-sweep --no-q80b > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_comb.csv
