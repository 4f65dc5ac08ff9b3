"""bench.py -- DynaExq hot path on B200: one step = one pass of the whole path over one decode batch
of the Qwen3-30B-A3B-shaped 48-layer MoE stack (BASELINE.json configs[1]):
per layer router logits -> top-k/gates/hotness counters -> permutation -> hybrid-precision expert
FFN over the slot pool -> combine, then the EMA fold, the periodic plan and the side-stream
promotions/demotions with their publication (DESIGN.md §1 rows a1-a14).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

Prints ONE JSON line (rank 0).  N > 1 (torchrun): expert parallelism (north_star) -- rank r
owns experts [r*E/N, (r+1)*E/N) of every layer with a per-GPU budget of 24e9/N B, serves its own batch of
B tokens (weak scaling: global batch N*B) and the library exchanges rows over NCCL inside dx_moe_step
(dx_pool_create_ep); value = all ranks' tokens / max time.  --replicas runs N independent full replicas.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer tokens/s decode+prefill at 1/2/4/8 B200; weight-byte HBM GB/s vs peak"
UNIT = "layer-tokens/s"

# C2: Qwen3-30B-A3B expert geometry, 24e9 B expert budget per GPU, bf16/int4.
PROF_EVERY = 7
C2 = dict(L=48, E=128, k=8, H=2048, I=768, g=128, high=16, low=4, budget=24 * 10**9, s=1,
          alpha=0.95, Tp=16, W=32, dwell=16, lag=4, zipf=1.2, drift=32, frac=0.25, n_top=24)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--layers", type=int, default=C2["L"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--router-scale", type=float, default=3.0)
    ap.add_argument("--budget-gb", type=float, default=0.0, help="override the 24 GB expert budget (sweeps)")
    ap.add_argument("--ffn-path", type=int, default=0, help="0 tcgen05 grouped GEMM, 1 mma.sync cross-check")
    ap.add_argument("--prefill-tokens", type=int, default=4096)
    ap.add_argument("--prefill-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-batch-sweep", action="store_true")
    ap.add_argument("--no-q80b", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent full replicas instead of EP")
    ap.add_argument("--no-teleport", action="store_true", help="skip the zero-cost-transition replay (switch cost)")
    ap.add_argument("--no-prefetch-leg", action="store_true", help="skip the f-1 cross-layer prefetch measurement")
    ap.add_argument("--per-layer-calls", action="store_true", help="one dx_moe_step call per layer instead of "
                    "dx_moe_step_layers per stack step")
    ap.add_argument("--ep-loopback", action="store_true",
                    help="N = 1: run the expert-parallel path on a one-rank NCCL communicator (tests the EP leg)")
    ap.add_argument("--switch-stress", action="store_true",
                    help="C5 (SURVEY 8(d)): one Q30B layer, n_hot swept 10%%..100%%, drift 0.5 every period; "
                         "prints the C5 JSON line instead of the main one")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled every 10 ms DURING the timed region through NVML (pynvml,
    nvidia_ml_py); falls back to `nvidia-smi -lms 100` when NVML is unavailable.  At least one sample is
    always taken (on entry)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")
    NAMES = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.samples = []            # (sm_mhz, max_mhz, set(reasons))
        self.nv = None
        self.stop = threading.Event()

    def _nvml_sample(self):
        nv, h = self.nv, self.h
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = {"sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap, "hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown}
        self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                             float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)),
                             {k for k, v in bits.items() if r & v}))

    def _nvml_loop(self):
        while not self.stop.wait(0.01):
            try:
                self._nvml_sample()
            except Exception:
                return

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.idx)
            self._nvml_sample()
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.t.join(timeout=1)
            try:
                self._nvml_sample()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for a, b, r in self.samples:
            sm.append(a)
            mx.append(b)
            reasons |= r
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for n, v in zip(self.NAMES, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


# ---------------------------------------------------------------------------------------- ours
def host_masters(seed, L, E, H, I, rank, world, experts=None):
    """bf16 masters of the whole stack in page-locked host memory (the paper's DRAM cache,
    PAPER.md:236).  Multi-rank replica runs share one /dev/shm copy; `experts` = (lo, n): only the global
    experts [lo, lo + n) of every layer (an expert-parallel rank's slice), pointers [L][n]."""
    import torch
    import synth
    n = 3 * I * H
    if experts is not None:
        lo, ne = experts
        arr = np.empty(L * ne * n, dtype=np.uint16)
        for l in range(L):
            for e in range(ne):
                synth.expert_master_into(seed, l, lo + e, H, I, arr[(l * ne + e) * n:(l * ne + e + 1) * n])
        rc = torch.cuda.cudart().cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
        if int(rc) != 0:
            raise RuntimeError(f"cudaHostRegister failed: {rc}")
        return arr, [arr.ctypes.data + i * n * 2 for i in range(L * ne)]
    total = L * E * n
    shm_ok = False
    if world > 1:
        import shutil
        try:   # one shared copy only if /dev/shm can hold it (container /dev/shm is often small)
            shm_ok = shutil.disk_usage("/dev/shm").free > total * 2 * 1.05 or \
                os.path.exists(f"/dev/shm/dx_masters_{seed}_{L}_{E}_{H}_{I}.bin")
        except OSError:
            shm_ok = False
        import torch.distributed as dist   # a collective decision: every rank takes the same branch
        flag = torch.tensor([1 if shm_ok else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        shm_ok = bool(flag.item())
    if shm_ok:
        path = f"/dev/shm/dx_masters_{seed}_{L}_{E}_{H}_{I}.bin"
        if rank == 0 and (not os.path.exists(path) or os.path.getsize(path) != total * 2):
            mm = np.memmap(path + ".tmp", dtype=np.uint16, mode="w+", shape=(total,))
            _fill(mm, seed, L, E, H, I)
            mm.flush()
            del mm
            os.replace(path + ".tmp", path)
        import torch.distributed as dist
        dist.barrier()
        arr = np.memmap(path, dtype=np.uint16, mode="r+", shape=(total,))
    else:
        arr = np.empty(total, dtype=np.uint16)
        _fill(arr, seed, L, E, H, I)
    rc = torch.cuda.cudart().cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
    if int(rc) != 0:
        raise RuntimeError(f"cudaHostRegister failed: {rc}")
    return arr, [arr.ctypes.data + i * n * 2 for i in range(L * E)]


def router_weights(seed, l, E, H, scale):
    """Router W_r of layer l: synth uniform(±1/sqrt(H)) scaled by `scale` (x W_r^T then has std
    ~0.58*scale per logit, a per-token spread comparable to the Gumbel noise of the trace recipe) and
    re-rounded to bf16."""
    import synth
    w = synth.router_bf16(seed, l, E, H)
    f = (w.astype(np.uint32) << 16).view(np.float32) * np.float32(scale)
    u = f.view(np.uint32)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16        # round to nearest even
    return u.astype(np.uint16)


def _fill(arr, seed, L, E, H, I):
    import synth
    n = 3 * I * H
    for l in range(L):
        for e in range(E):
            synth.expert_master_into(seed, l, e, H, I, arr[(l * E + e) * n:(l * E + e + 1) * n])


def run_ours(a, rank, world, local_rank):
    import torch
    import synth
    from paper_2511_15015_b200 import dx
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    c = dict(C2)
    L, E, k, H, I, g, B = a.layers, c["E"], c["k"], c["H"], c["I"], c["g"], a.batch
    seed = a.seed
    ep_mode = (world > 1 and not a.replicas) or a.ep_loopback
    G = world if ep_mode else 1
    E_loc = E // G
    if ep_mode:       # the batch-sweep / prefill legs are single-GPU studies
        a.no_batch_sweep, a.prefill_tokens = True, 0
    t0 = time.time()
    arr, ptrs = host_masters(seed, L, E, H, I, rank, world, experts=(rank * E_loc, E_loc) if ep_mode else None)
    t_gen = time.time() - t0
    cfg = dx.dx_config()
    cfg.num_layers, cfg.num_experts, cfg.top_k, cfg.hidden, cfg.inter, cfg.group_size = L, E, k, H, I, g
    cfg.high_bits, cfg.low_bits = c["high"], c["low"]
    budget = int(a.budget_gb * 1e9) if a.budget_gb > 0 else c["budget"]
    cfg.expert_budget_bytes = budget * L // C2["L"] // G         # per GPU: the north_star's artificial budget
    cfg.n_spare, cfg.ema_alpha = c["s"], c["alpha"]
    cfg.period, cfg.warmup_steps, cfg.dwell_min, cfg.publish_lag = c["Tp"], c["W"], c["dwell"], c["lag"]
    cfg.max_tokens, cfg.ep_rank, cfg.ep_size = max(B, 64, a.prefill_tokens), rank if ep_mode else 0, G
    stream = torch.cuda.current_stream()
    nccl_id = None
    if ep_mode:       # the library's own NCCL communicator; its id travels over torch.distributed
        import torch.distributed as dist
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(dx.dx_get_unique_id()), dtype=torch.uint8))
        if world > 1:
            dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().tolist())
    t0 = time.time()
    pool = dx.Pool(cfg, ptrs, stream, nccl_id=nccl_id)
    t_pool = time.time() - t0
    n_hot = pool.info.n_hot
    if a.ffn_path:
        pool.dx_set_ffn_path(a.ffn_path)
    # router weights per layer + Zipf bias per (layer, drift epoch) -> skewed, drifting routing
    wr = torch.empty(L, E, H, dtype=torch.bfloat16, device=dev)
    for l in range(L):
        wr[l].copy_(torch.from_numpy(router_weights(seed, l, E, H, a.router_scale).view(np.int16)).view(torch.bfloat16))
    total_steps = c["W"] + a.warmup + 2 * a.steps + 2
    n_epochs = total_steps // c["drift"] + 2
    bias = torch.empty(L, n_epochs, E, dtype=torch.float32, device=dev)
    for l in range(L):
        for ep in range(n_epochs):
            rk = synth.rank_perm(seed, l, ep, E, c["n_top"], c["frac"])
            bias[l, ep].copy_(torch.from_numpy(synth.zipf_logp(rk, c["zipf"])))
    xs_host = torch.empty(total_steps, B, H, dtype=torch.int16, pin_memory=True)
    for s_ in range(total_steps):
        xs_host[s_].copy_(torch.from_numpy(synth.normal_bf16(seed, 100 + rank, s_, 0, (B, H)).view(np.int16)))
    xs = xs_host.to(dev).view(torch.bfloat16)
    y = torch.empty(2, B, H, dtype=torch.bfloat16, device=dev)
    step_counter = [0]

    # raw device pointers, as a C/C++ caller of the ABI would hold them (no per-call tensor indexing)
    y_p = [y[i].data_ptr() for i in range(2)]
    wr_p = [wr[l].data_ptr() for l in range(L)]
    bias_p = [[bias[l, ep].data_ptr() for ep in range(n_epochs)] for l in range(L)]
    nonlocal_pool = [pool]             # the pool step() drives (the teleport replay swaps in its own)
    P = dx.Pool.ptr_array
    y_arr = P([y_p[l & 1] for l in range(L)])
    wr_arr = P(wr_p)
    bias_arr = [P([bias_p[l][ep] for l in range(L)]) for ep in range(n_epochs)]
    x_arr_cache = {}

    def step(x):
        s_ = step_counter[0]
        ep = s_ // c["drift"]
        xp = x if isinstance(x, int) else x.data_ptr()
        if a.per_layer_calls:
            mstep = nonlocal_pool[0].dx_moe_step   # forward + hotness update + plan, fold fused into the combine
            for l in range(L):
                mstep(l, xp, B, y_p[l & 1], router_w=wr_p[l], router_bias=bias_p[l][ep])
        else:                                      # the whole stack step in one C call (dx_moe_step per layer)
            xa = x_arr_cache.get(xp)
            if xa is None:
                xa = x_arr_cache[xp] = P([xp] * L)
            nonlocal_pool[0].dx_moe_step_layers(0, L, xa, B, y_arr, router_w_arr=wr_arr, router_bias_arr=bias_arr[ep])
        step_counter[0] += 1

    # controller warm-up (t < W) and finalize at t = W, then the bench warm-up
    def warm(pool_):
        for s_ in range(c["W"]):
            step(xs[s_])
        for l in range(L):
            pool_.dx_plan_precision(l)
        for s_ in range(a.warmup):
            step(xs[c["W"] + s_])
        pool_.dx_sync()

    warm(pool)
    pool.dx_profile_read()
    dist_on = world > 1
    if dist_on:
        import torch.distributed as dist
    # ---------------- timed region (device-resident inputs)
    base = c["W"] + a.warmup
    # CUDA-event timing of every PROF_EVERY-th forward (7: coprime with the 48 layers, so the samples
    # rotate over all of them; the host cost of event records stays off the other forwards)
    pool.dx_profile_enable(PROF_EVERY)
    launches0 = pool.dx_kernel_launches()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        h0 = time.perf_counter()
        for s_ in range(a.steps):
            step(xs[base + s_])
        host_ms = (time.perf_counter() - h0) * 1e3      # host issue time of the timed steps (no sync inside)
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = pool.dx_kernel_launches() - launches0
    prof = pool.dx_profile_read()
    pool.dx_profile_enable(False)
    ms_max = ms
    if dist_on:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_max = float(tt.item())

    # host cost of issuing one stack step into an empty launch queue (the timed region's host time is paced by the
    # GPU once the queue is full, so it measures the GPU, not the host)
    host_one = []
    for s_ in range(5):
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        step(xs[base + s_])
        host_one.append((time.perf_counter() - h0) * 1e3)
    torch.cuda.synchronize()

    def teleport_replay():
        """The same steps from a fresh pool whose transitions are free (dx_set_teleport): identical routing,
        plans and per-step tier tables, no transfer work -- SURVEY §8(d)'s exposed switch time is
        (t_on - t_teleport) / t_on over the timed steps."""
        tp = dx.Pool(cfg, ptrs, stream, nccl_id=None)
        tp.dx_set_teleport(True)
        saved = step_counter[0]
        step_counter[0] = 0
        nonlocal_pool[0] = tp
        warm(tp)
        tp.dx_profile_enable(PROF_EVERY)           # the same event sampling as the timed run
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s_ in range(a.steps):
            step(xs[base + s_])
        e1.record(stream)
        torch.cuda.synchronize()
        nonlocal_pool[0] = pool
        step_counter[0] = saved
        tp.close()
        return e0.elapsed_time(e1)
    # ---------------- end-to-end: host x -> device, stack, y -> host, every step
    e2e = None
    if not a.no_e2e:
        yh = torch.empty(B, H, dtype=torch.bfloat16, pin_memory=True)
        xdev = torch.empty(B, H, dtype=torch.bfloat16, device=dev)
        base2 = base + a.steps
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s_ in range(a.steps):
            xdev.view(torch.int16).copy_(xs_host[base2 + s_], non_blocking=True)
            step(xdev)
            yh.copy_(y[(L - 1) & 1], non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        if dist_on:
            tt = torch.tensor([e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        e2e = {"value": world * B * L * a.steps / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": B * H * 2, "d2h_bytes_per_step": B * H * 2, "ms_per_step": e_ms / a.steps}
    peak, peak_src = load_peaks()
    scale = L * a.steps / max(prof["forwards"], 1)     # all forwards / event-timed (sampled) forwards
    wb = prof["weight_bytes"]
    ffn_ms = prof["ffn_ms"]
    ach0 = wb[0] / (ffn_ms[0] / 1e3) / 1e9 if ffn_ms[0] > 0 else 0.0
    ach_all = (wb[0] + wb[1]) / ((ffn_ms[0] + ffn_ms[1]) / 1e3) / 1e9
    fused = prof.get("ffn_fused", 0) > 0     # decode FFN as ONE launch: the roofline kernel covers both phases
    rf_kernel = ("k_gemm<2,1> fused decode FFN: gate/up + SwiGLU, then down + gate scaling, one persistent launch "
                 "(tcgen05)") if fused else "k_gemm<0> decode gate/up + SwiGLU (tcgen05)"
    rf_ach = ach_all if fused else ach0
    rf_bytes = (wb[0] + wb[1]) if fused else wb[0]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ffn_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:     # measured DRAM bytes per launch of the same kernel (one ncu --set full capture)
            traffic = json.load(f).get("fused_dram_bytes_per_launch" if fused else "gateup_dram_bytes_per_launch")
    out = {
        "metric": METRIC, "value": world * B * L * a.steps / (ms_max / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded splitmix64 weights, "
        "Zipf(1.2) router bias with drift; see DESIGN.md input recipe)",
        "config": {"workload": f"C2: Qwen3-30B-A3B-shaped {L}-layer MoE decode stack (E=128, top-8, H=2048, "
                               f"I=768), batch {B} per GPU, {budget / 1e9 / G:g}e9 B expert budget per GPU "
                               f"(n_hot={n_hot}/{E_loc} bf16, rest int4 g=128), router mode (W_r x{a.router_scale:g} "
                               "+ Zipf(1.2) bias, ~90 experts touched per layer), controller Tp=16 L=4 with drift"
                               + (f"; expert parallel over {G} GPUs (NCCL all-to-all inside libdx)" if ep_mode else ""),
                   "global_batch": B * world,
                   "parallelism": f"ep{G}" if ep_mode else (f"replicas x{world}" if world > 1 else "single"),
                   "l2": "no flush: each step streams >=48 distinct layers of weights (> 126 MB L2)"},
        "roofline": {"bound": "hbm", "kernel": rf_kernel, "achieved": rf_ach, "peak": peak,
                     "unit": "GB/s", "frac": rf_ach / peak, "traffic": traffic, "peak_source": peak_src,
                     "ffn_both_phases_gbs": ach_all, "ffn_both_frac": ach_all / peak,
                     # the whole layer (routing, both GEMMs, combine, fold, plan periods, switching): every touched
                     # expert's algorithmic weight bytes over the device time of the whole timed stack
                     "layer_achieved": (wb[0] + wb[1]) / max(prof["forwards"], 1) * L * a.steps / (ms / 1e3) / 1e9,
                     "layer_frac": (wb[0] + wb[1]) / max(prof["forwards"], 1) * L * a.steps / (ms / 1e3) / 1e9 / peak,
                     "algorithmic_bytes_per_launch": rf_bytes / max(prof["forwards"], 1)},
        "gpu_launches": launches,
        "e2e": e2e,
        "extra": {"ffn_ms_share": (ffn_ms[0] + ffn_ms[1]) * scale / ms if ms > 0 else None,
                  "fwd_ms_share": prof["fwd_ms"] * scale / ms if ms > 0 else None,
                  "profiled_forwards": prof["forwards"], "forwards": L * a.steps,
                  "active_experts_per_layer": prof["active_experts"] / max(prof["forwards"], 1),
                  "weight_bytes_per_layer": (wb[0] + wb[1]) / max(prof["forwards"], 1),
                  "route_ms_share": prof["route_ms"] * scale / ms if ms > 0 else None,
                  "switch": {"plans": prof["plans"], "promotions": prof["promotions"],
                             "demotions": prof["demotions"], "publishes": prof["publishes"],
                             "exposed_ms_total": prof["exposed_ms"],
                             "exposed_frac_of_step_time": prof["exposed_ms"] / ms if ms > 0 else None,
                             "xfer_ms_mean": prof["xfer_ms"] / max(prof["plans"], 1),
                             "promotion_gbs": prof["copy_bytes"] / (prof["copy_ms"] / 1e3) / 1e9
                             if prof["copy_ms"] > 0 else None,
                             "xfer_ms_max": prof["xfer_max_ms"]},
                  "setup_s": {"masters": t_gen, "pool_create": t_pool},
                  "host_issue_ms_per_step": host_ms / a.steps,
                  "host_issue_note": "timed-region issue time; paced by the GPU once the launch queue is full",
                  "host_cost_ms_per_step": statistics.median(host_one),
                  "host_cost_note": "median host time to issue one stack step into an empty launch queue (5 samples)"},
    }
    clock = clk.summary()
    if clock:
        out["clocks"] = clock
    if not a.no_batch_sweep:
        out["extra"]["decode_batch_sweep"] = batch_sweep(a, pool, wr, bias, step_counter, L, H, dev, stream, peak)
    if not a.no_batch_sweep:
        out["extra"]["zipf_sweep"] = zipf_sweep(a, pool, wr, step_counter, L, E, H, dev, stream, peak)
    if a.prefill_tokens > 0:
        out["extra"]["prefill"] = prefill_leg(a, pool, wr, bias, step_counter, L, E, H, I, k, c, dev, stream)
    pool.close()
    if not ep_mode and not a.no_batch_sweep:
        out["extra"]["tier_brackets"] = tier_brackets(a, cfg, ptrs, L, E, H, B, dev, stream, peak, wr_arr, bias_arr)
    if not ep_mode and not a.no_prefetch_leg:
        out["extra"]["prefetch"] = prefetch_leg(a, ptrs, L, E, k, H, I, g, c, dev, stream)
    if not ep_mode and not a.no_teleport:
        ms_tel = teleport_replay()
        sw = out["extra"]["switch"]
        sw["teleport_ms_per_step"] = ms_tel / a.steps
        sw["on_ms_per_step"] = ms / a.steps
        sw["exposed_frac_teleport"] = (ms - ms_tel) / ms
        sw["definition"] = ("(t_on - t_teleport) / t_on over the timed steps; teleport = a fresh pool replaying the "
                            "same steps with dx_set_teleport (same plans and tier tables, no transfers)")
    torch.cuda.cudart().cudaHostUnregister(arr.ctypes.data)
    del arr
    return out


def c4_ep_local_leg(a, peak, L=4):
    """C4 on ONE GPU: the Qwen3-Next-80B-A3B-shaped layer (E=512, top-10, H=2048, I=512, g=128, int4
    HIGH / int2 LOW) partitioned over G in {1, 2, 4, 8} ranks with C4's per-GPU budgets (n_hot = 25 % of E_loc, s = 1:
    543.6 / 273.0 / 137.8 / 70.1 MB per layer per rank), every rank's pool in this process (a local EP group: the
    library's EP layer with the deduplicated exchange done by device copies), B = 64 tokens per rank, router mode with
    a drifting Zipf(1.2) bias, 10 timed steps after the warm-up and finalize.  All ranks share the one GPU, so this is
    not a scaling curve: it measures the EP layer's correctness-path cost, the per-rank weight bytes and the
    deduplication at each G (the multi-GPU curve is bench.py --gpus N under torchrun)."""
    import torch
    import synth
    from paper_2511_15015_b200 import dx
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    E, k, H, I, g, hb, lb, s_sp, B = 512, 10, 2048, 512, 128, 4, 2, 1, 64
    seed = a.seed + 3
    arr, ptrs = host_masters(seed, L, E, H, I, 0, 1)
    S_h, S_l = dx.dx_slot_bytes(H, I, g, hb), dx.dx_slot_bytes(H, I, g, lb)
    wr = torch.stack([torch.from_numpy(router_weights(seed, l, E, H, a.router_scale).view(np.int16)).view(torch.bfloat16)
                      for l in range(L)]).to(dev)
    out = {"workload": f"C4 on one GPU: {L}-layer Qwen3-Next-80B-A3B-shaped stack (E=512, top-10, I=512, int4/int2), "
                       f"G ranks' pools as a local EP group, B={B} per rank, per-rank budget n_hot = 25 % of E/G, s=1"}
    for G in (1, 2, 4, 8):
        e_loc = E // G
        n_hot = e_loc // 4
        M = n_hot * S_h + (e_loc - n_hot) * S_l + s_sp * (S_h + S_l)
        pools = []
        for r in range(G):
            cfg = dx.dx_config()
            cfg.num_layers, cfg.num_experts, cfg.top_k, cfg.hidden, cfg.inter, cfg.group_size = L, E, k, H, I, g
            cfg.high_bits, cfg.low_bits = hb, lb
            cfg.expert_budget_bytes = M * L
            cfg.n_spare, cfg.ema_alpha = s_sp, 0.95
            cfg.period, cfg.warmup_steps, cfg.dwell_min, cfg.publish_lag = 16, 32, 16, 4
            cfg.max_tokens, cfg.ep_rank, cfg.ep_size = B, r, G
            rp = [ptrs[l * E + r * e_loc + e] for l in range(L) for e in range(e_loc)]
            pools.append(dx.Pool(cfg, rp, stream, nccl_id=b"local"))
        bias = [torch.stack([torch.from_numpy(synth.zipf_logp(synth.rank_perm(seed, l, ep, E, 128, 0.25), 1.2))
                             for ep in range(4)]).to(dev) for l in range(L)]
        xs = [[torch.from_numpy(synth.normal_bf16(seed, 960 + r, i, 0, (B, H)).view(np.int16)).to(dev).view(torch.bfloat16)
               for i in range(2)] for r in range(G)]
        ys = [torch.empty(B, H, dtype=torch.bfloat16, device=dev) for _ in range(G)]
        cnt = [0]

        def st():
            ep = min(cnt[0] // 16, 3)
            for l in range(L):
                dx.dx_moe_step_group(pools, l, [xs[r][cnt[0] & 1] for r in range(G)], [B] * G, ys,
                                     router_w=[wr[l]] * G, router_bias=[bias[l][ep]] * G)
            cnt[0] += 1

        for _ in range(32):
            st()
        for l in range(L):
            for p in pools:
                p.dx_plan_precision(l)
        for _ in range(3):
            st()
        for p in pools:
            p.dx_sync()
            p.dx_profile_read()
            p.dx_profile_enable(True)
        t0 = [p.dx_ep_traffic() for p in pools]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n = 10
        for _ in range(n):
            st()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        prof = [p.dx_profile_read() for p in pools]
        t1 = [p.dx_ep_traffic() for p in pools]
        rows = sum(b["rows_sent"] - a_["rows_sent"] for a_, b in zip(t0, t1))
        ents = sum(b["entries_sent"] - a_["entries_sent"] for a_, b in zip(t0, t1))
        wb = sum(pr["weight_bytes"][0] + pr["weight_bytes"][1] for pr in prof)
        fw = sum(pr["forwards"] for pr in prof)
        out[f"G{G}"] = {"per_rank_budget_mb": M / 1e6, "n_hot_per_rank": n_hot, "value": G * B * L * n / (ms / 1e3),
                        "unit": UNIT, "ms_per_step": ms / n, "x_rows_sent": rows, "dispatch_entries": ents,
                        "dedup_factor": ents / max(rows, 1), "weight_bytes_per_rank_layer": wb / max(fw, 1)}
        for p in pools:
            p.close()
    torch.cuda.cudart().cudaHostUnregister(arr.ctypes.data)
    return out


def prefetch_leg(a, ptrs, L_all, E, k, H, I, g, c, dev, stream, L=8):
    """f-1: an 8-layer C2-shaped stack (the first 8 layers' masters, C2's per-layer
    budget -> n_hot 24) in trace mode with cross-layer-coupled routing (synth.coupled_trace_logits: layer l boosts
    pi_l of layer l-1's choices; Zipf(1.2) with a quarter of the top-24 set drifting every 16 steps), B = 64,
    Tp=16, L=4, run from fresh pools on identical inputs: cross-layer prefetch off, then on with fan-out 1 and 2
    (lead 4); and f-4, the same run with the HIGH images on the SSD tier behind a 16-image DRAM cache.  Per run over the last 48 steps (3 plan periods): promotions, prefetch hits, mean side-stream switch
    time per plan (issue -> ready), copy-engine bytes per plan and the device ms per step."""
    import torch
    import synth
    from paper_2511_15015_b200 import dx
    B, Tp, W, lag, steps_timed = 64, 16, 32, 4, 48
    total = W + 8 + steps_timed
    lgs = torch.empty(total, L, B, E, dtype=torch.float32, device=dev)
    for s_ in range(total):
        ls = synth.coupled_trace_logits(a.seed + 7, L, s_, B, E, k, 6.0, 1.2, 16, 0.25, 24)
        for l in range(L):
            lgs[s_, l].copy_(torch.from_numpy(ls[l]))
    xs = torch.from_numpy(synth.normal_bf16(a.seed, 950, 0, 0, (2, B, H)).view(np.int16)).to(dev).view(torch.bfloat16)
    y = torch.empty(L, B, H, dtype=torch.bfloat16, device=dev)
    res = {"workload": f"f-1: {L}-layer C2-shaped stack, trace mode with cross-layer coupled routing (boost 6 on "
                       f"pi_l of layer l-1's top-{k}), drift 25 % of the top-24 set every 16 steps, B={B}, Tp={Tp}, "
                       f"L={lag}; lead 4; last {steps_timed} steps"}
    for mode, fan in (("off", 0), ("on_f1", 1), ("on_f2", 2), ("ssd_tier", 0)):
        cfg = dx.dx_config()
        cfg.num_layers, cfg.num_experts, cfg.top_k, cfg.hidden, cfg.inter, cfg.group_size = L, E, k, H, I, g
        cfg.high_bits, cfg.low_bits = c["high"], c["low"]
        cfg.expert_budget_bytes = c["budget"] * L // c["L"]
        cfg.n_spare, cfg.ema_alpha = c["s"], c["alpha"]
        cfg.period, cfg.warmup_steps, cfg.dwell_min, cfg.publish_lag = Tp, W, Tp, lag
        cfg.max_tokens, cfg.ep_rank, cfg.ep_size = B, 0, 1
        if mode == "ssd_tier":       # f-4: HIGH images in a file on the box's disk behind a 16-image DRAM cache
            pool = dx.Pool(cfg, ptrs[:L * E], stream, ssd_path=os.path.join("/tmp", f"dx_bench_ssd_{os.getpid()}.bin"),
                           dram_cache_images=16)
        else:
            pool = dx.Pool(cfg, ptrs[:L * E], stream)
        if fan:
            pool.dx_set_prefetch(fan, 4)
        P = pool.ptr_array
        x_arr = [P([xs[i]] * L) for i in range(2)]
        y_arr = P([y[l] for l in range(L)])

        def st(s_):
            pool.dx_moe_step_layers(0, L, x_arr[s_ & 1], B, y_arr, logits_arr=P([lgs[s_, l] for l in range(L)]))

        for s_ in range(total - steps_timed):
            st(s_)
        pool.dx_sync()
        pool.dx_profile_read()
        pool.dx_profile_enable(PROF_EVERY)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s_ in range(total - steps_timed, total):
            st(s_)
        e1.record(stream)
        pool.dx_sync()
        ms = e0.elapsed_time(e1)
        pr = pool.dx_profile_read()
        pool.close()
        res[mode] = {"ms_per_step": ms / steps_timed, "plans": pr["plans"], "promotions": pr["promotions"],
                     "prefetch_issued": pr["prefetch_issued"], "prefetch_hits": pr["prefetch_hits"],
                     "switch_ms_mean": pr["xfer_ms"] / max(pr["plans"], 1),
                     "copy_mb_per_plan": pr["copy_bytes"] / max(pr["plans"], 1) / 1e6}
        if mode == "ssd_tier":
            res[mode].update({"ssd_reads": pr["ssd_reads"], "ssd_mb": pr["ssd_bytes"] / 1e6,
                              "ssd_read_gbs": pr["ssd_bytes"] / (pr["ssd_read_ms"] / 1e3) / 1e9 if pr["ssd_read_ms"] > 0
                              else None, "dram_cache_hits": pr["dram_cache_hits"]})
    for m in ("on_f1", "on_f2"):
        res[m]["hit_rate"] = res[m]["prefetch_hits"] / max(res[m]["promotions"], 1)
    return res


def q80b_leg(a, peak, L=8):
    """C4's layer shape on one GPU: a Qwen3-Next-80B-A3B-shaped stack (E=512, top-10,
    H=2048, I=512, g=128) with the paper's int4 (HIGH) / int2 (LOW) pair, the per-GPU budget
    of C4 at G=1 (n_hot = 25 % of E, s = 1 -> 543.6 MB per layer), router mode with a drifting Zipf(1.2)
    bias.  Decode B=64 and prefill T=4096: layer-tokens/s, the expert GEMMs' weight GB/s (decode) and
    TFLOP/s (prefill).  L=8 layers (per-layer numbers; 48 layers of bf16 masters would not fit host RAM
    next to C2's)."""
    import torch
    import synth
    from paper_2511_15015_b200 import dx
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    E, k, H, I, g, hb, lb, s_sp = 512, 10, 2048, 512, 128, 4, 2, 1
    seed = a.seed + 1
    arr, ptrs = host_masters(seed, L, E, H, I, 0, 1)
    S_h, S_l = dx.dx_slot_bytes(H, I, g, hb), dx.dx_slot_bytes(H, I, g, lb)
    n_hot = E // 4
    M = n_hot * S_h + (E - n_hot) * S_l + s_sp * (S_h + S_l)
    cfg = dx.dx_config()
    cfg.num_layers, cfg.num_experts, cfg.top_k, cfg.hidden, cfg.inter, cfg.group_size = L, E, k, H, I, g
    cfg.high_bits, cfg.low_bits = hb, lb
    cfg.expert_budget_bytes = M * L
    cfg.n_spare, cfg.ema_alpha = s_sp, 0.95
    cfg.period, cfg.warmup_steps, cfg.dwell_min, cfg.publish_lag = 16, 32, 16, 4
    cfg.max_tokens, cfg.ep_rank, cfg.ep_size = 4096, 0, 1
    cfg.n_shared = 1                  # Qwen3-Next's shared expert (f-3, Eq. 1's first sum), int4 like the HIGH tier
    sh = np.empty(L * 3 * I * H, dtype=np.uint16)
    for l in range(L):
        synth.expert_master_into(seed + 1, l, 0, H, I, sh[l * 3 * I * H:(l + 1) * 3 * I * H])
    torch.cuda.cudart().cudaHostRegister(sh.ctypes.data, sh.nbytes, 0)
    pool = dx.Pool(cfg, ptrs + [sh.ctypes.data + l * 3 * I * H * 2 for l in range(L)], stream)
    assert pool.info.n_hot == n_hot, (pool.info.n_hot, n_hot)
    wr = torch.empty(L, E, H, dtype=torch.bfloat16, device=dev)
    for l in range(L):
        wr[l].copy_(torch.from_numpy(router_weights(seed, l, E, H, a.router_scale).view(np.int16)).view(torch.bfloat16))
    n_ep = 8
    bias = torch.empty(L, n_ep, E, dtype=torch.float32, device=dev)
    for l in range(L):
        for ep in range(n_ep):
            bias[l, ep].copy_(torch.from_numpy(synth.zipf_logp(synth.rank_perm(seed, l, ep, E, n_hot, 0.25), 1.2)))
    res = {"workload": f"C4 shape at G=1: {L}-layer Qwen3-Next-80B-A3B-shaped stack (E=512, top-10, H=2048, I=512, "
                       f"one shared expert per layer at the HIGH tier), "
                       f"int4 HIGH / int2 LOW g=128, n_hot={n_hot} (25 %), s=1, {M / 1e6:.1f} MB per layer"}
    cnt = [0]
    for name, T, n_t in (("decode", 64, 10), ("prefill", 4096, 2)):
        xs = [torch.from_numpy(synth.normal_bf16(seed, 600 + T, i, 0, (T, H)).view(np.int16)).to(dev).view(torch.bfloat16)
              for i in range(2)]
        y = torch.empty(T, H, dtype=torch.bfloat16, device=dev)

        def qstep(x):
            ep = min(cnt[0] // 32, n_ep - 1)
            for l in range(L):
                pool.dx_moe_step(l, x, T, y, router_w=wr[l], router_bias=bias[l, ep])
            cnt[0] += 1

        if name == "decode":
            for i in range(32):
                qstep(xs[i % 2])
            for l in range(L):
                pool.dx_plan_precision(l)
        for i in range(3):
            qstep(xs[i % 2])
        pool.dx_sync()
        pool.dx_profile_read()
        pool.dx_profile_enable(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(n_t):
            qstep(xs[i % 2])
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        prof = pool.dx_profile_read()
        pool.dx_profile_enable(False)
        ffn_s = (prof["ffn_ms"][0] + prof["ffn_ms"][1]) / 1e3
        wb = prof["weight_bytes"][0] + prof["weight_bytes"][1]
        r = {"value": T * L * n_t / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / n_t, "steps": n_t,
             "active_experts_per_layer": prof["active_experts"] / max(prof["forwards"], 1),
             "weight_bytes_per_layer": wb / max(prof["forwards"], 1)}
        if name == "decode":
            r["ffn_weight_gbs"] = wb / ffn_s / 1e9 if ffn_s > 0 else 0.0
            r["ffn_hbm_frac"] = r["ffn_weight_gbs"] / peak
        else:
            r["gemm_tflops"] = 2.0 * T * (k + 1) * 3 * I * H * prof["forwards"] / ffn_s / 1e12 if ffn_s > 0 else 0.0
        res[name] = r
    pool.close()
    torch.cuda.cudart().cudaHostUnregister(arr.ctypes.data)
    torch.cuda.cudart().cudaHostUnregister(sh.ctypes.data)
    return res


def batch_sweep(a, pool, wr, bias, step_counter, L, H, dev, stream, peak):
    """C2's decode batch range (B in 1..64) on the same stack and pool: per B, 5 timed
    stack steps (after 2 untimed) -> layer-tokens/s, and the expert GEMMs' algorithmic weight bytes /
    their device time (both phases) against the HBM peak."""
    import torch
    import synth
    c = C2
    rows = []
    for B in (1, 2, 4, 8, 16, 32, 64):
        xs = [torch.from_numpy(synth.normal_bf16(a.seed, 800 + B, i, 0, (B, H)).view(np.int16)).to(dev).view(torch.bfloat16)
              for i in range(2)]
        y = torch.empty(B, H, dtype=torch.bfloat16, device=dev)
        P = pool.ptr_array
        y_arr, wr_arr = P([y] * L), P([wr[l] for l in range(L)])
        x_arrs = {x.data_ptr(): P([x] * L) for x in xs}
        b_arrs = [P([bias[l, e_] for l in range(L)]) for e_ in range(bias.shape[1])]

        def bstep(x):
            ep = min(step_counter[0] // c["drift"], bias.shape[1] - 1)
            pool.dx_moe_step_layers(0, L, x_arrs[x.data_ptr()], B, y_arr, router_w_arr=wr_arr, router_bias_arr=b_arrs[ep])
            step_counter[0] += 1

        for i in range(2):
            bstep(xs[i % 2])
        pool.dx_sync()
        pool.dx_profile_read()
        pool.dx_profile_enable(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n = 5
        for i in range(n):
            bstep(xs[i % 2])
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        prof = pool.dx_profile_read()
        pool.dx_profile_enable(False)
        wb = prof["weight_bytes"][0] + prof["weight_bytes"][1]
        ffn_s = (prof["ffn_ms"][0] + prof["ffn_ms"][1]) / 1e3
        gbs = wb / ffn_s / 1e9 if ffn_s > 0 else 0.0
        rows.append({"batch": B, "value": B * L * n / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / n,
                     "active_experts_per_layer": prof["active_experts"] / max(prof["forwards"], 1),
                     "weight_bytes_per_layer": wb / max(prof["forwards"], 1), "ffn_weight_gbs": gbs,
                     "ffn_hbm_frac": gbs / peak})
    return rows


def zipf_sweep(a, pool, wr, step_counter, L, E, H, dev, stream, peak):
    """SURVEY §8(d) C2 routing skew s in {0, 0.8, 1.2} (the bench's main line is 1.2): B = 64 decode on the same
    stack and pool (HIGH set as the controller left it), 5 timed steps per s after 2 untimed; layer-tokens/s, touched
    experts and the expert GEMMs' weight GB/s."""
    import torch
    import synth
    B, rows = 64, []
    xs = [torch.from_numpy(synth.normal_bf16(a.seed, 870, i, 0, (B, H)).view(np.int16)).to(dev).view(torch.bfloat16)
          for i in range(2)]
    y = torch.empty(B, H, dtype=torch.bfloat16, device=dev)
    P = pool.ptr_array
    y_arr, wr_arr = P([y] * L), P([wr[l] for l in range(L)])
    x_arrs = [P([x] * L) for x in xs]
    for s in (0.0, 0.8, 1.2):
        bias = torch.stack([torch.from_numpy(synth.zipf_logp(synth.rank_perm(a.seed, l, 0, E, 24, 0.25), s))
                            for l in range(L)]).to(dev)
        b_arr = P([bias[l] for l in range(L)])
        for i in range(2):
            pool.dx_moe_step_layers(0, L, x_arrs[i % 2], B, y_arr, router_w_arr=wr_arr, router_bias_arr=b_arr)
            step_counter[0] += 1
        pool.dx_sync()
        pool.dx_profile_read()
        pool.dx_profile_enable(True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n = 5
        for i in range(n):
            pool.dx_moe_step_layers(0, L, x_arrs[i % 2], B, y_arr, router_w_arr=wr_arr, router_bias_arr=b_arr)
            step_counter[0] += 1
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        prof = pool.dx_profile_read()
        pool.dx_profile_enable(False)
        wb = prof["weight_bytes"][0] + prof["weight_bytes"][1]
        ffn_s = (prof["ffn_ms"][0] + prof["ffn_ms"][1]) / 1e3
        gbs = wb / ffn_s / 1e9 if ffn_s > 0 else 0.0
        rows.append({"zipf_s": s, "value": B * L * n / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / n,
                     "active_experts_per_layer": prof["active_experts"] / max(prof["forwards"], 1),
                     "weight_bytes_per_layer": wb / max(prof["forwards"], 1), "ffn_weight_gbs": gbs,
                     "ffn_hbm_frac": gbs / peak})
    return rows


def tier_brackets(a, cfg0, ptrs, L, E, H, B, dev, stream, peak, wr_arr, bias_arr):
    """The uniform brackets of the C2 decode line: every expert at bf16 (budget for n_hot = E) and
    every expert at int4 (n_hot = 0), fresh pools over the same stack and inputs, router mode, 10 timed steps after
    the warm-up and finalize; layer-tokens/s and the expert GEMMs' weight GB/s against the HBM peak."""
    import ctypes
    import torch
    import synth
    from paper_2511_15015_b200 import dx
    S_h, S_l = dx.dx_slot_bytes(H, cfg0.inter, cfg0.group_size, 16), dx.dx_slot_bytes(H, cfg0.inter, cfg0.group_size, 4)
    s_sp = cfg0.n_spare
    out = {}
    xs = [torch.from_numpy(synth.normal_bf16(a.seed, 880, i, 0, (B, H)).view(np.int16)).to(dev).view(torch.bfloat16)
          for i in range(2)]
    y = torch.empty(2, B, H, dtype=torch.bfloat16, device=dev)
    for name, n_hot in (("all_bf16", E), ("all_int4", 0)):
        cfg = dx.dx_config()
        ctypes.memmove(ctypes.addressof(cfg), ctypes.addressof(cfg0), ctypes.sizeof(cfg))
        cfg.expert_budget_bytes = L * (n_hot * S_h + (E - n_hot) * S_l + s_sp * (S_h + S_l))
        pool = dx.Pool(cfg, ptrs, stream)
        assert pool.info.n_hot == n_hot, (pool.info.n_hot, n_hot)
        P = pool.ptr_array
        y_arr = P([y[l & 1] for l in range(L)])
        x_arrs = [P([x] * L) for x in xs]

        def st(i):
            pool.dx_moe_step_layers(0, L, x_arrs[i & 1], B, y_arr, router_w_arr=wr_arr, router_bias_arr=bias_arr[0])

        for i in range(cfg.warmup_steps):
            st(i)
        for l in range(L):
            pool.dx_plan_precision(l)
        for i in range(3):
            st(i)
        pool.dx_sync()
        pool.dx_profile_read()
        pool.dx_profile_enable(PROF_EVERY)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n = 10
        for i in range(n):
            st(i)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        prof = pool.dx_profile_read()
        pool.close()
        wb = prof["weight_bytes"][0] + prof["weight_bytes"][1]
        ffn_s = (prof["ffn_ms"][0] + prof["ffn_ms"][1]) / 1e3
        g0 = (prof["weight_bytes"][0] / (prof["ffn_ms"][0] / 1e3) / 1e9
              if prof["ffn_ms"][0] > 0 and not prof.get("ffn_fused", 0) else None)
        gbs = wb / ffn_s / 1e9 if ffn_s > 0 else 0.0
        out[name] = {"n_hot": n_hot, "value": B * L * n / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / n,
                     "weight_bytes_per_layer": wb / max(prof["forwards"], 1), "gateup_gbs": g0, "gateup_frac": g0 / peak if g0 is not None else None,
                     "ffn_weight_gbs": gbs, "ffn_hbm_frac": gbs / peak}
    return out


def prefill_leg(a, pool, wr, bias, step_counter, L, E, H, I, k, c, dev, stream):
    """C3: 4k-token prefill steps over the same stack and pool (drifting routing, the
    controller keeps planning and transitioning).  Reports layer-tokens/s and the expert GEMMs'
    tensor-pipe utilisation (FLOPs = 2*T*k*3*I*H per layer) against the measured bf16 peak."""
    import torch
    import synth
    T = a.prefill_tokens
    xs = [torch.from_numpy(synth.normal_bf16(a.seed, 900, i, 0, (T, H)).view(np.int16)).to(dev).view(torch.bfloat16)
          for i in range(2)]
    y = torch.empty(T, H, dtype=torch.bfloat16, device=dev)

    def pstep(x):
        ep = step_counter[0] // c["drift"]
        for l in range(L):
            pool.dx_moe_step(l, x, T, y, router_w=wr[l], router_bias=bias[l, min(ep, bias.shape[1] - 1)])
        step_counter[0] += 1

    for i in range(2):
        pstep(xs[i % 2])
    pool.dx_sync()
    pool.dx_profile_read()
    pool.dx_profile_enable(True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(a.prefill_steps):
        pstep(xs[i % 2])
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    prof = pool.dx_profile_read()
    pool.dx_profile_enable(False)
    flops_layer = 2.0 * T * k * 3 * I * H
    gemm_ms = prof["ffn_ms"][0] + prof["ffn_ms"][1]
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    peak_tf = float(peaks.get("bf16_tflops", 1590.0))
    tf = flops_layer * prof["forwards"] / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    return {"workload": f"C3: {L}-layer stack, T={T} tokens per step, same pool/controller",
            "value": T * L * a.prefill_steps / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / a.prefill_steps,
            "steps": a.prefill_steps, "gemm_tflops": tf, "tensor_peak_tflops": peak_tf,
            "tensor_frac": tf / peak_tf, "gemm_ms_share": gemm_ms / ms,
            "weight_bytes_per_layer": sum(prof["weight_bytes"]) / max(prof["forwards"], 1)}


def switch_stress(a):
    """C5: one Qwen3-30B-A3B-shaped layer (E=128, bf16/int4, s=2 spares per tier) at
    n_hot = 10 %..100 % of E, with the hot set drifting (half of the top-n_hot set rotates every period),
    so the controller promotes and demotes every period.  Per n_hot and per workload (decode B=16,
    prefill T=4096): device ms per step, transitions, side-stream switch latency (plan issue -> ready,
    CUDA events on the side stream) and EXPOSED switch time = compute-stream stall at publication
    (events around the cross-stream wait), as a fraction of the step time."""
    import torch
    import synth
    from paper_2511_15015_b200 import dx
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    E, k, H, I, g, s_sp = 128, 8, 2048, 768, 128, 2
    W, alpha = 16, 0.9
    # publish lag sized so the lag window (lag x step time) covers a plan's transfers (~0.5-1 ms: a 9.4 MB
    # promotion over PCIe plus a demotion): decode steps of one layer take ~0.11 ms, prefill steps ~1 ms
    lag_of = {"decode": (16, 10), "prefill": (8, 2)}          # mode -> (Tp, L)
    arr, ptrs = host_masters(a.seed, 1, E, H, I, 0, 1)
    S_h, S_l = dx.dx_slot_bytes(H, I, g, 16), dx.dx_slot_bytes(H, I, g, 4)
    wr = torch.from_numpy(router_weights(a.seed, 0, E, H, a.router_scale).view(np.int16)).to(dev).view(torch.bfloat16)
    stream = torch.cuda.current_stream()
    rows = []
    for n_hot in (13, 26, 38, 51, 64, 77, 90, 102, 115, 128):
        budget = n_hot * S_h + (E - n_hot) * S_l + s_sp * (S_h + S_l)
        for mode, T, steps in (("decode", 16, 64), ("prefill", 4096, 24)):
            Tp, lag = lag_of[mode]
            cfg = dx.dx_config()
            cfg.num_layers, cfg.num_experts, cfg.top_k, cfg.hidden, cfg.inter, cfg.group_size = 1, E, k, H, I, g
            cfg.high_bits, cfg.low_bits = 16, 4
            cfg.expert_budget_bytes = budget
            cfg.n_spare, cfg.ema_alpha = s_sp, alpha
            cfg.period, cfg.warmup_steps, cfg.dwell_min, cfg.publish_lag = Tp, W, Tp, lag
            cfg.max_tokens, cfg.ep_rank, cfg.ep_size = T, 0, 1
            total = W + Tp + steps + 1
            bias = torch.stack([torch.from_numpy(synth.zipf_logp(
                synth.rank_perm(a.seed, 0, ep, E, max(n_hot, 1), 0.5), 1.2)) for ep in range(total // Tp + 2)]).to(dev)
            xs = [torch.from_numpy(synth.normal_bf16(a.seed, 700, i, 0, (T, H)).view(np.int16)).to(dev).view(torch.bfloat16)
                  for i in range(2)]
            y = torch.empty(T, H, dtype=torch.bfloat16, device=dev)

            def run_cfg(teleport):
                pool = dx.Pool(cfg, ptrs, stream)
                assert pool.info.n_hot == n_hot, (pool.info.n_hot, n_hot)
                pool.dx_set_teleport(teleport)

                def one(t):
                    pool.dx_moe_forward(0, xs[t & 1], T, y, router_w=wr, router_bias=bias[t // Tp])
                    pool.dx_hotness_update(0)
                    pool.dx_plan_precision(0)

                for t in range(W):
                    one(t)
                pool.dx_plan_precision(0)
                for t in range(W, W + Tp):
                    one(t)
                pool.dx_sync()
                pool.dx_profile_read()
                pool.dx_profile_enable(True)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for t in range(W + Tp, W + Tp + steps):
                    one(t)
                e1.record(stream)
                torch.cuda.synchronize()
                ms_ = e0.elapsed_time(e1)
                pr_ = pool.dx_profile_read()
                pool.dx_profile_enable(False)
                pool.close()
                return ms_, pr_

            ms, pr = run_cfg(False)
            ms_tel, _ = run_cfg(True)
            rows.append({"n_hot": n_hot, "hot_frac": n_hot / E, "mode": mode, "tokens": T, "steps": steps,
                         "ms_per_step": ms / steps, "teleport_ms_per_step": ms_tel / steps,
                         "exposed_frac_teleport": (ms - ms_tel) / ms if ms > 0 else None,
                         "promotions": pr["promotions"], "demotions": pr["demotions"],
                         "plans": pr["plans"], "switch_ms_mean": pr["xfer_ms"] / max(pr["plans"], 1),
                         "switch_ms_max": pr["xfer_max_ms"], "Tp": Tp, "publish_lag": lag,
                         "promotion_gbs": pr["copy_bytes"] / (pr["copy_ms"] / 1e3) / 1e9 if pr["copy_ms"] > 0 else None,
                         "publish_stall_ms": pr["exposed_ms"],
                         "publish_stall_frac": pr["exposed_ms"] / ms if ms > 0 else None})
    torch.cuda.cudart().cudaHostUnregister(arr.ctypes.data)
    return {"metric": "C5 precision-switch stress: exposed switch time (t_on - t_teleport) / t_on", "unit": "fraction",
            "higher_is_better": False, "n_gpus": 1, "data": "synthetic",
            "config": {"workload": "C5: one Q30B-shaped layer (E=128, k=8, H=2048, I=768, bf16/int4 g=128), "
                                   "s=2 spares per tier, W=16, dwell=Tp, alpha=0.9, decode B=16 (Tp=16, L=10) and "
                                   "prefill T=4096 (Tp=8, L=2), Zipf(1.2) router bias with half of the top-n_hot set "
                                   "rotating every period"},
            "value": max(r["exposed_frac_teleport"] for r in rows), "rows": rows}


# ---------------------------------------------------------------------------------------- oracle arm
def oracle_layer_sample(a, seconds=15.0, max_steps=None):
    """The CPU oracle (as it stands) on a bounded sample of the same workload: one layer of the stack
    (layer 0), batch B, router mode, controller fold/plan, FFN from pre-dequantised stable images."""
    import oracle
    import synth
    c = dict(C2)
    E, k, H, I, g, B = c["E"], c["k"], c["H"], c["I"], c["g"], a.batch
    n_hot = oracle.n_hot(c["budget"] // c["L"], E, oracle.slot_bytes(H, I, g, 16), oracle.slot_bytes(H, I, g, 4),
                         c["s"])
    wr = router_weights(a.seed, 0, E, H, a.router_scale)
    rk = synth.rank_perm(a.seed, 0, 0, E, c["n_top"], c["frac"])
    bias = synth.zipf_logp(rk, c["zipf"])
    tiers = {e: bool(rk[e] < n_hot) for e in range(E)}
    ctrl = oracle.Controller(E, n_hot, c["s"], c["alpha"], c["Tp"], 0, c["dwell"], c["lag"])
    ctrl.plan()
    Wcache = {}
    nthreads = os.cpu_count() or 1
    times = []
    t_start = time.time()
    s_ = 0
    while True:
        x = synth.normal_bf16(a.seed, 100, s_, 0, (B, H))
        lg = oracle.router_logits(x, wr, bias).astype(np.float32)
        idx, gate = oracle.route(lg, k)
        for e in np.unique(idx):          # stable images prepared outside the timed part (as the pool is)
            e = int(e)
            if e not in Wcache:
                Wcache[e] = oracle.expert_tier(synth.expert_master(a.seed, 0, e, H, I), H, I, g, 16, 4, tiers[e])
        t0 = time.perf_counter()
        lg = oracle.router_logits(x, wr, bias).astype(np.float32)
        idx, gate = oracle.route(lg, k)
        _, y = oracle.moe_ffn(x, idx, gate, Wcache, H, I, nthreads=nthreads)
        _, mass = oracle.counts(idx, gate, E)
        ctrl.fold(mass, B)
        ctrl.plan()
        times.append(time.perf_counter() - t0)
        s_ += 1
        if (max_steps and s_ >= max_steps) or (not max_steps and sum(times) >= seconds) or \
                time.time() - t_start > 4 * seconds:
            break
    return B / statistics.mean(times), nthreads, len(times), times


def oracle_extra_timings(a):
    """SURVEY §8(d)'s oracle timing plan beside the main cpu_baseline (the oracle as it stands, host cores):
    C1 in full (300 steps: route, counters, fold, plan, FFN), the group quantiser on one Q30B expert, one plan at
    E = 512, and one C3 layer (T = 4096, top-8) estimated from a bounded 64-token sample of it."""
    import oracle
    import synth
    out = {"cores": os.cpu_count() or 1}
    # C1 in full
    E, k, H, I, g, T = 8, 2, 64, 128, 32, 32
    W = {e: oracle.expert_tier(synth.expert_master(a.seed, 0, e, H, I), H, I, g, 16, 4, e < 2) for e in range(E)}
    ctrl = oracle.Controller(E, 2, 1, 0.9, 8, 16, 16, 2)
    t0 = time.perf_counter()
    for step in range(300):
        lg = synth.trace_logits(a.seed, 0, step, T, E, 1.2, 16, 0.5, 2)
        idx, gate = oracle.route(lg, k)
        oracle.moe_ffn(synth.normal_bf16(a.seed, 1, step, 0, (T, H)), idx, gate, W, H, I)
        ctrl.fold(oracle.counts(idx, gate, E)[1], T)
        ctrl.plan()
    out["c1_300_steps_s"] = time.perf_counter() - t0
    # quantiser on one Q30B expert (3 matrices of 768 x 2048, int4, g = 128)
    m = synth.expert_master(a.seed, 0, 0, 2048, 768)
    t0 = time.perf_counter()
    oracle.expert_tier(m, 2048, 768, 128, 16, 4, False)
    out["quantize_q30b_expert_s"] = time.perf_counter() - t0
    # one plan at E = 512
    c512 = oracle.Controller(512, 128, 1, 0.95, 16, 1, 16, 4)
    rng = np.random.default_rng(0)
    c512.fold(rng.integers(0, 1 << 24, 512, dtype=np.uint64), 64)
    c512.plan()                                   # finalize
    for _ in range(15):
        c512.fold(rng.integers(0, 1 << 24, 512, dtype=np.uint64), 64)
        c512.plan()
    c512.fold(rng.integers(0, 1 << 24, 512, dtype=np.uint64), 64)
    t0 = time.perf_counter()
    c512.plan()
    out["plan_e512_s"] = time.perf_counter() - t0
    # C3: one T = 4096 layer from a 64-token sample
    E, k, H, I = 128, 8, 2048, 768
    lg = synth.trace_logits(a.seed, 0, 0, 64, E, 1.2)
    idx, gate = oracle.route(lg, k)
    Wc = {int(e): oracle.expert_tier(synth.expert_master(a.seed, 0, int(e), H, I), H, I, 128, 16, 4, int(e) % 5 == 0)
          for e in np.unique(idx)}
    x = synth.normal_bf16(a.seed, 2, 0, 0, (64, H))
    t0 = time.perf_counter()
    oracle.moe_ffn(x, idx, gate, Wc, H, I, nthreads=os.cpu_count() or 1)
    dt = time.perf_counter() - t0
    out["c3_layer_est_s"] = dt * 4096 / 64
    out["c3_sample"] = "64 of the 4096 tokens (top-8 FFN over pre-dequantised images, all host threads), scaled x64"
    return out


def run_reference(a, rank, world):
    if rank != 0:
        return None
    n = a.warmup + a.steps
    val, cores, nsteps, times = oracle_layer_sample(a, max_steps=n)
    t = times[a.warmup:] if len(times) > a.warmup else times
    v = a.batch / statistics.mean(t)
    sample = f"layer 0 of the C2 stack, batch {a.batch}, {len(t)} timed steps (router, top-k, FFN, fold, plan)"
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * statistics.mean(t), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C2 layer sample, batch {a.batch}", "global_batch": a.batch},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    a = parse()
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() in ("VERSION", ""):
        os.environ["NCCL_DEBUG"] = "WARN"        # NCCL's version banner would precede the one JSON line on stdout
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if a.impl == "ours":
            torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl" if a.impl == "ours" else "gloo")
    if a.impl == "reference":
        out = run_reference(a, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:                      # the other ranks load libdx.so only once rank 0 has (re)built it
        import torch.distributed as dist
        dist.barrier()
    if a.switch_stress:
        if rank == 0:
            print(json.dumps(switch_stress(a)), flush=True)
        return
    out = run_ours(a, rank, world, local_rank)
    if rank == 0 and world == 1 and not a.no_q80b:
        out["extra"]["q80b"] = q80b_leg(a, out["roofline"]["peak"])
        out["extra"]["c4_ep_local"] = c4_ep_local_leg(a, out["roofline"]["peak"])
    if rank == 0:
        if not a.no_cpu_baseline and world == 1:          # the oracle baseline is an N = 1 figure
            v, cores, nsteps, _ = oracle_layer_sample(a, seconds=15.0)
            out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                   "sample": f"layer 0 of the C2 stack, batch {a.batch}, {nsteps} steps "
                                             "(router, top-k, FFN over pre-dequantised stable images, fold, plan)"}
            if not a.no_batch_sweep:
                out["cpu_baseline"]["extra_timings"] = oracle_extra_timings(a)
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
