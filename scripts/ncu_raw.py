"""Key metrics from an ncu report's raw page: python scripts/ncu_raw.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
extra = [x for x in sys.argv[2:]]
for r in data:
    print("---")
    for w in want + extra:
        if w in h:
            i = h.index(w)
            print(f"  {w:70s} {r[i]} {units[i]}")
