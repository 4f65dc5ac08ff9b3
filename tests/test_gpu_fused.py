"""The launch-structure choices do not change results: the fused decode FFN launch (k_gemm<2,1>, DX_FUSE) and the
wide prefill tiles of the bf16 experts (k_wide, DX_WIDE) compute every output entry with the same K order as the split
launches, so a layer's outputs are bitwise equal either way.  Each variant runs in its own process (the switches are
read once per process)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import hashlib, os, sys
sys.path.insert(0, os.environ["DX_ROOT"]); sys.path.insert(0, os.path.join(os.environ["DX_ROOT"], "tests"))
import numpy as np, torch, synth
from dxtest import Masters, bf16_dev, budget_for, make_cfg
from paper_2511_15015_b200 import dx
E, k, H, I, g = 32, 4, 256, 128, 64
m = Masters(11, 1, E, H, I)
cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, 8, 1), 1, 0.9, 4, 1, 4, 1, 512)
pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
h = hashlib.sha256()
for step, T in enumerate([32, 48, 300, 17, 512, 64]):   # decode (T <= 64) and prefill sizes, HIGH bf16 after step 0
    lg = torch.from_numpy(synth.trace_logits(11, 0, step, T, E, 1.2)).cuda()
    x = bf16_dev(synth.normal_bf16(11, 1, step, 0, (T, H)))
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    pool.dx_moe_step(0, x, T, y, logits=lg)
    torch.cuda.synchronize()
    h.update(y.view(torch.int16).cpu().numpy().tobytes())
print(pool.dx_get_table(0)["tier"].sum(), h.hexdigest())
pool.close()
"""


def _run(env_extra):
    env = dict(os.environ, DX_ROOT=ROOT, **env_extra)
    out = subprocess.run([sys.executable, "-c", SNIPPET], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.gpu
def test_fused_and_wide_launches_are_bitwise_the_split_ones():
    base = _run({"DX_FUSE": "0", "DX_WIDE": "0"})
    n_hot, _ = base.split()
    assert int(n_hot) > 0, "the layer must have HIGH (bf16) experts for k_wide to run"
    assert _run({"DX_FUSE": "1", "DX_WIDE": "0"}) == base
    assert _run({"DX_FUSE": "0", "DX_WIDE": "1"}) == base
    assert _run({"DX_FUSE": "1", "DX_WIDE": "1"}) == base
