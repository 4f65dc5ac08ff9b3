"""Host-side cost of each ABI call in the C2 decode step (no syncs inside the loop): where the ~125 us of
host issue time per layer goes."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import synth
from paper_2511_15015_b200 import dx

L, E, k, H, I, g, B = 8, 128, 8, 2048, 768, 128, 64
arr, ptrs = bench.host_masters(0, L, E, H, I, 0, 1)
cfg = dx.dx_config()
cfg.num_layers, cfg.num_experts, cfg.top_k, cfg.hidden, cfg.inter, cfg.group_size = L, E, k, H, I, g
cfg.high_bits, cfg.low_bits = 16, 4
cfg.expert_budget_bytes = 24 * 10**9 * L // 48
cfg.n_spare, cfg.ema_alpha = 1, 0.95
cfg.period, cfg.warmup_steps, cfg.dwell_min, cfg.publish_lag = 16, 32, 16, 4
cfg.max_tokens, cfg.ep_rank, cfg.ep_size = 64, 0, 1
pool = dx.Pool(cfg, ptrs, torch.cuda.current_stream())
wr = torch.randn(L, E, H, device="cuda").bfloat16() * 0.02
bias = torch.zeros(E, device="cuda")
x = torch.randn(B, H, device="cuda").bfloat16()
y = torch.empty(B, H, device="cuda", dtype=torch.bfloat16)
xp, yp, bp = x.data_ptr(), y.data_ptr(), bias.data_ptr()
wp = [wr[l].data_ptr() for l in range(L)]
for s in range(40):
    for l in range(L):
        pool.dx_moe_forward(l, xp, B, yp, router_w=wp[l], router_bias=bp)
        pool.dx_hotness_update(l)
        pool.dx_plan_precision(l)
torch.cuda.synchronize()
tf = th = tp = 0.0
n = 30
for s in range(n):
    for l in range(L):
        t0 = time.perf_counter(); pool.dx_moe_forward(l, xp, B, yp, router_w=wp[l], router_bias=bp)
        t1 = time.perf_counter(); pool.dx_hotness_update(l)
        t2 = time.perf_counter(); pool.dx_plan_precision(l)
        t3 = time.perf_counter()
        tf += t1 - t0; th += t2 - t1; tp += t3 - t2
torch.cuda.synchronize()
c = n * L
print(f"host us per call: forward {1e6 * tf / c:.1f}, hotness {1e6 * th / c:.1f}, plan {1e6 * tp / c:.1f}")
# ctypes floor: a call that returns immediately
t0 = time.perf_counter()
for i in range(10000):
    dx.dx_version()
print(f"ctypes floor {1e6 * (time.perf_counter() - t0) / 10000:.2f} us")
# raw launch cost: empty torch op
t0 = time.perf_counter()
for i in range(1000):
    y.zero_()
torch.cuda.synchronize()
print(f"torch zero_ launch {1e6 * (time.perf_counter() - t0) / 1000:.2f} us")
pool.dx_set_ffn_path(1)
tf = 0.0
for s in range(n):
    for l in range(L):
        t0 = time.perf_counter(); pool.dx_moe_forward(l, xp, B, yp, router_w=wp[l], router_bias=bp)
        tf += time.perf_counter() - t0
        pool.dx_hotness_update(l)
        pool.dx_plan_precision(l)
torch.cuda.synchronize()
print(f"host us per forward with the mma.sync FFN path (small kernel params): {1e6 * tf / c:.1f}")
pool.close()
