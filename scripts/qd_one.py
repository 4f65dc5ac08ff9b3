"""One Q30B layer decode forward, repeated: gate/up and down GB/s from the pool's event timing (dx_profile).
python scripts/qd_one.py n_hot B zipf [reps]   (n_hot 0 = all int4, 128 = all bf16).  Used for k_qdec tuning and
under ncu (one layer, so the captured launches are the same expert set)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from dxtest import Masters, bf16_dev, budget_for, make_cfg  # noqa: E402
from paper_2511_15015_b200 import dx  # noqa: E402

E, k, H, I, g = 128, 8, 2048, 768, 128
n_hot, B, zipf = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 200
L = 4                              # > L2 between repeats
m = Masters(1, L, E, H, I)
cfg = make_cfg(dx, L, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, n_hot, 1, L), 1, 0.95, 16, 1, 32, 4, 256)
pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
x0 = synth.normal_bf16(1, 0, 0, 0, (64, H))
y = torch.zeros(64, H, dtype=torch.bfloat16, device="cuda")
lg0 = synth.trace_logits(1, 0, 0, 64, E, 1.2)
for layer in range(L):
    pool.dx_moe_forward(layer, bf16_dev(x0), 64, y, logits=torch.from_numpy(lg0).cuda())
    pool.dx_hotness_update(layer)
    pool.dx_plan_precision(layer)  # finalize: the n_hot hottest go HIGH
lg = torch.from_numpy(synth.trace_logits(1, 0, 5, B, E, zipf)).cuda()
xd = bf16_dev(synth.normal_bf16(1, 0, 5, 0, (B, H)))
yd = torch.zeros(B, H, dtype=torch.bfloat16, device="cuda")
kw = dict(logits=lg)
if os.environ.get("QD_ROUTER"):                 # router mode (the bench's): logits = x W_r^T + b on the device
    gen = torch.Generator(device="cuda").manual_seed(7)
    wr = (torch.randn(E, H, device="cuda", generator=gen) / H ** 0.5).to(torch.bfloat16)
    rb = torch.log(torch.arange(1, E + 1, device="cuda", dtype=torch.float32) ** -max(zipf, 1e-3))
    kw = dict(router_w=wr, router_bias=rb)
for i in range(10):
    pool.dx_moe_forward(i % L, xd, B, yd, **kw)
pool.dx_profile_enable(1)
for i in range(reps):
    pool.dx_moe_forward(i % L, xd, B, yd, **kw)
pr = pool.dx_profile_read()
n = pr["forwards"]
gu, dn = pr["ffn_ms"][0] / n, pr["ffn_ms"][1] / n
bg, bd = pr["weight_bytes"][0] / n, pr["weight_bytes"][1] / n
print(f"n_hot {n_hot} B {B} zipf {zipf}: active {pr['active_experts'] / n:.1f}  gate/up {gu * 1e3:.1f} us {bg / gu / 1e6:.0f} GB/s"
      f"  down {dn * 1e3:.1f} us {bd / dn / 1e6:.0f} GB/s  fwd {pr['fwd_ms'] / n * 1e3:.1f} us")
pool.close()
