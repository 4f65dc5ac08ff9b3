set -x
nproc; free -g | head -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -s 25000 -c 1200 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
