"""GPU test of f-4, the SSD tier ("high- and low-precision weights are stored on SSD and cached in
DRAM"): a pool whose HIGH images live in a library-written file behind a small pinned DRAM cache
(dx_pool_create_ssd) must behave bit for bit like the plain pool (HIGH images in pinned DRAM) over warm-up, the
finalize (initial HIGH set read through the cache), plan periods with promotions and demotions, and a manual
promotion: every layer output bitwise, the controller tables equal, and the exported HIGH images of promoted experts
bit-exact against the oracle's canonical images; with a cache smaller than the working set every promotion of a new
image really reads the file (the read count and bytes are reported)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from dxtest import Masters, bf16_dev, budget_for, canon_expected, make_cfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_15015_b200 import dx as _dx
    return _dx


@pytest.mark.parametrize("pair", [(16, 4), (4, 2)], ids=["bf16-int4", "int4-int2"])
def test_ssd_tier_matches_dram_pool(dx, pair, tmp_path):
    hb, lb = pair
    E, k, H, I, g, T, n_hot = 16, 4, 256, 128, 64, 24, 4
    Tp, W, lag = 4, 6, 1
    m = Masters(17, 1, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, hb, lb, budget_for(E, H, I, g, hb, lb, n_hot, 1), 1, 0.8, Tp, W, Tp, lag, T)
    path = str(tmp_path / f"dx_ssd_{os.getpid()}.bin")
    ssd = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream(), ssd_path=path, dram_cache_images=2)
    assert os.path.getsize(path) > 0
    plain = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    ssd.dx_profile_enable(True)
    for step in range(40):
        x = bf16_dev(synth.normal_bf16(17, 1, step, 0, (T, H)))
        lg = torch.from_numpy(synth.trace_logits(17, 0, step, T, E, 1.2, 8, 0.5, n_hot)).cuda()
        ys, yp = (torch.zeros(T, H, dtype=torch.bfloat16, device="cuda") for _ in range(2))
        ssd.dx_moe_step(0, x, T, ys, logits=lg)
        plain.dx_moe_step(0, x, T, yp, logits=lg)
        assert torch.equal(ys.view(torch.int16), yp.view(torch.int16)), step
        ts, tp = ssd.dx_get_table(0), plain.dx_get_table(0)
        for key in ("tier", "slot", "version", "in_flight"):
            assert np.array_equal(ts[key], tp[key]), (step, key)
    # a manual promotion through the SSD tier too
    ssd.dx_sync()
    plain.dx_sync()
    low = [e for e in range(E) if ssd.dx_get_table(0)["tier"][e] == 0][:1]
    occ = ssd.dx_occupancy(0)
    if low and occ["cap_hi"] > occ["used_hi"]:
        assert ssd.dx_promote(0, low) == plain.dx_promote(0, low)
        ssd.dx_sync()
        plain.dx_sync()
    tab = ssd.dx_get_table(0)
    for e in range(E):
        if tab["tier"][e] == 1 and tab["version"][e] > 0:
            img = ssd.dx_export_expert(0, e)
            assert np.array_equal(img, canon_expected(m.get(0, e), H, I, g, hb, lb, True)), e
    pr = ssd.dx_profile_read()
    print(f"SSD tier {pair}: {pr['ssd_reads']} reads ({pr['ssd_bytes'] / 1e6:.2f} MB, {pr['ssd_read_ms']:.2f} ms), "
          f"{pr['dram_cache_hits']} cache hits, versions {int(tab['version'].sum())}")
    assert int(tab["version"].sum()) > n_hot                       # transitions after the finalize happened
    assert pr["ssd_reads"] > 0 and pr["ssd_bytes"] == pr["ssd_reads"] * (ssd.info.export_bytes_hi if hb == 16 else
                                                                          ssd.info.slot_bytes_hi)
    ssd.close()
    plain.close()
    assert not os.path.exists(path)                                # the library removes its file


def test_ssd_tier_bad_path(dx):
    E, k, H, I, g = 8, 2, 64, 128, 32
    m = Masters(18, 1, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, 2, 1), 1, 0.9, 8, 4, 8, 2, 16)
    with pytest.raises(dx.DxError):
        dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream(), ssd_path="/nonexistent_dir/x.bin", dram_cache_images=2)
    with pytest.raises(dx.DxError):
        dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream(), ssd_path="/tmp/x.bin", dram_cache_images=0)
