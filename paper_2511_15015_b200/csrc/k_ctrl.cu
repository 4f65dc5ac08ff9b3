// k_ctrl.cu -- the precision controller on the device (a10, a11), side-stream transitions
// (a12 demotion, a13 promotion) and publication (a14).
//   Eq. 2 EMA hotness; Alg. 1 UpdateHotness/PrecisionSchedule;
//   §3.3 asynchronous promotion/demotion, registration, "last stable version";
//   §3.4 fixed-block pools, immediate reclaim; §3.5 tau_h.
// Readings R-H2 (fp64 EMA, no FMA), R-C1..R-C4 (plan), R-P3 (warm-up finalize), R-T1 (publish).
// The plan runs on the device so the whole controller is host-sync free; the host only knows the
// deterministic schedule (when a plan / publish is due), never the plan contents.
#include "dx_quant.cuh"

#define CTRL_THREADS 1024

namespace {

__device__ __forceinline__ int32_t bscan_excl(int32_t v, int32_t* tmp, int32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) tmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int32_t s = lane < nw ? tmp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) tmp[lane] = s;
    }
    __syncthreads();
    const int32_t r = (warp > 0 ? tmp[warp - 1] : 0) + x - v;
    *total = tmp[nw - 1];
    __syncthreads();
    return r;
}

// ------------------------------------------------------------------ a10 + a14
__global__ void __launch_bounds__(CTRL_THREADS) k_fold(Ctrl c, int layer, u64 B_tot, double oma) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    fold_layer(c, layer, B_tot, oma);
}

// ------------------------------------------------------------------ a11
__global__ void __launch_bounds__(CTRL_THREADS) k_plan(Ctrl c, int layer, int finalize) {
    __shared__ double Ss[CTRL_THREADS];
    __shared__ int32_t order[CTRL_THREADS];
    __shared__ int32_t freelist[CTRL_THREADS];
    __shared__ int32_t tmp[32];
    __shared__ int32_t any_pending;
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int E = c.E, s = c.s, n_hot = c.n_hot;
    const int tid = threadIdx.x;
    const int base = layer * E, ob = layer * (E + s);
    const i64 t = c.t[layer];
    int32_t* lo_own = c.lo_owner + ob;
    int32_t* hi_own = c.hi_owner + ob;
    int4* plan = c.plan_cmd + base;
    if (tid == 0) any_pending = 0;
    for (int e = tid; e < CTRL_THREADS; e += blockDim.x) Ss[e] = e < E ? c.S[base + e] : 0.0;
    __syncthreads();
    // rank under (S desc, id asc)
    int32_t rank = 0;
    const int e = tid;
    if (e < E) {
        const double se = Ss[e];
        for (int j = 0; j < E; ++j) {
            const double sj = Ss[j];
            rank += (sj > se) || (sj == se && j < e);
        }
        order[rank] = e;
    }
    __syncthreads();
    int32_t total;
    if (finalize) {
        const bool hot = e < E && rank < n_hot;
        const int cap_lo = E - n_hot + s, cap_hi = n_hot + s;
        if (tid == 0) {
            c.tau[layer] = n_hot <= 0 ? __longlong_as_double(0x7ff0000000000000LL)
                         : (n_hot >= E ? __longlong_as_double((long long)0xfff0000000000000ULL)
                                       : Ss[order[n_hot - 1]]);
            c.cap_lo[layer] = cap_lo;
            c.cap_hi[layer] = cap_hi;
        }
        for (int i = tid; i < E + s; i += blockDim.x) { lo_own[i] = -1; hi_own[i] = -1; }
        __syncthreads();
        int32_t my_slot = e < E ? c.slot[base + e] : 0;
        if (e < E && !hot && my_slot < cap_lo) lo_own[my_slot] = e;
        __syncthreads();
        const bool mover = e < E && !hot && my_slot >= cap_lo;
        int32_t nm;
        const int32_t mi = bscan_excl(mover ? 1 : 0, tmp, &nm);
        const bool fr = tid < cap_lo && lo_own[tid] < 0;
        int32_t nf;
        const int32_t fi = bscan_excl(fr ? 1 : 0, tmp, &nf);
        if (fr) freelist[fi] = tid;
        __syncthreads();
        if (mover) {
            const int d = freelist[mi];
            lo_own[d] = e;
            plan[mi] = make_int4(e, 0, d, my_slot);
            c.slot[base + e] = d;
        }
        if (hot) {
            hi_own[rank] = e;
            plan[nm + rank] = make_int4(e, 1, rank, my_slot);
            c.tier[base + e] = 1;
            c.slot[base + e] = rank;
            c.version[base + e] += 1;
            c.last[base + e] = t;
        }
        if (tid == 0) c.plan_n[layer] = nm + n_hot;
        return;
    }
    // regular period: nothing may be in flight (else deferred, R-C2)
    if (e < E && c.pend_dir[base + e] != 0) any_pending = 1;
    __syncthreads();
    if (any_pending) {
        if (tid == 0) c.plan_n[layer] = 0;
        return;
    }
    const double tau = c.tau[layer];
    const int cap_lo = c.cap_lo[layer], cap_hi = c.cap_hi[layer];
    // flags indexed by rank r = tid
    bool pf = false, df = false;
    int32_t er = -1;
    if (tid < E) {
        er = order[tid];
        const int i = base + er;
        const bool inH = (tid < n_hot) && (Ss[er] >= tau);
        const bool dw = (t - c.last[i]) >= c.dwell;
        pf = inH && c.tier[i] == 0 && dw;
        df = !inH && c.tier[i] == 1 && dw;
    }
    int32_t nP, nD, nHigh, nfl, nfh;
    const int32_t ppos = bscan_excl(pf ? 1 : 0, tmp, &nP);
    const int32_t dpos_fwd = bscan_excl(df ? 1 : 0, tmp, &nD);
    const int32_t dpos = df ? (nD - 1 - dpos_fwd) : 0;           // descending rank order
    bscan_excl((tid < E && c.tier[base + tid] == 1) ? 1 : 0, tmp, &nHigh);
    const bool frl = tid < cap_lo && lo_own[tid] < 0;
    const int32_t fl = bscan_excl(frl ? 1 : 0, tmp, &nfl);
    if (frl) freelist[fl] = tid;
    __syncthreads();
    const int32_t nd = nD < nfl ? nD : nfl;
    if (df && dpos < nd) {
        const int i = base + er;
        const int d = freelist[dpos];
        lo_own[d] = er;
        plan[dpos] = make_int4(er, -1, d, c.slot[i]);
        c.pend_dir[i] = -1; c.pend_dst[i] = d; c.pend_at[i] = t + c.lag; c.last[i] = t;
    }
    __syncthreads();
    const bool frh = tid < cap_hi && hi_own[tid] < 0;
    const int32_t fh = bscan_excl(frh ? 1 : 0, tmp, &nfh);
    if (frh) freelist[fh] = tid;
    __syncthreads();
    int32_t np = nP < nfh ? nP : nfh;
    const int32_t capn = n_hot - nHigh + nd;
    if (np > capn) np = capn;
    if (np < 0) np = 0;
    if (pf && ppos < np) {
        const int i = base + er;
        const int d = freelist[ppos];
        hi_own[d] = er;
        plan[nd + ppos] = make_int4(er, 1, d, c.slot[i]);
        c.pend_dir[i] = 1; c.pend_dst[i] = d; c.pend_at[i] = t + c.lag; c.last[i] = t;
    }
    if (tid == 0) {
        c.plan_n[layer] = nd + np;
        if (c.tstats) { c.tstats[0] += (u64)np; c.tstats[1] += (u64)nd; }
    }
}

// ------------------------------------------------------------------ manual commands (host-chosen)
// status per command: 0 ok, 1 wrong tier / not ready, 2 range, 4 exhausted, 5 busy
__global__ void k_manual(Ctrl c, int layer, const int2* __restrict__ cmds, int n, int32_t* __restrict__ status) {
    if (threadIdx.x != 0) return;
    const int E = c.E, base = layer * E, ob = layer * (E + c.s);
    const i64 t = c.t[layer];
    int np = 0;
    for (int q = 0; q < n; ++q) {
        const int e = cmds[q].x, dir = cmds[q].y;
        int st = 0;
        if (e < 0 || e >= E || (dir != 1 && dir != -1)) st = 2;
        else if (c.pend_dir[base + e]) st = 5;
        else if ((dir > 0) == (c.tier[base + e] == 1)) st = 1;
        else {
            int32_t* own = dir > 0 ? c.hi_owner + ob : c.lo_owner + ob;
            const int cap = dir > 0 ? c.cap_hi[layer] : c.cap_lo[layer];
            int d = -1;
            for (int j = 0; j < cap; ++j) if (own[j] < 0) { d = j; break; }
            if (d < 0) st = 4;
            else {
                own[d] = e;
                const int i = base + e;
                c.plan_cmd[base + np++] = make_int4(e, dir, d, c.slot[i]);
                c.pend_dir[i] = dir; c.pend_dst[i] = d; c.pend_at[i] = t + c.lag; c.last[i] = t;
            }
        }
        status[q] = st;
    }
    c.plan_n[layer] = np;
}

// ------------------------------------------------------------------ a12 / a13 / relayout moves
// Persistent grid over (command, chunk).  Promotion: stream the HIGH image from pinned host memory
// (zero-copy over PCIe, no SM-side staging) into the destination HIGH block.  Demotion: group-
// quantise the current HIGH block into the destination LOW block on the device (R-Q2).  Moves
// (finalize only): LOW block -> LOW block.
#define XFER_CHUNKS 64
// mode: 0 = regular plan (promotions + demotions), 1 = finalize moves only, 2 = finalize promotions
// only (the second finalize pass runs after every move has left the future HIGH region), 3 = demotions only
// (runtime plans: the promotions' H2D copies run on the copy engine, issued by the host).
// Side-stream transitions run as a few small, register-lean blocks (128 threads, <= 48 registers) so
// that each fits on an SM next to a resident persistent k_gemm CTA (736 threads x 80 registers): the
// transfer then overlaps the expert GEMMs instead of holding SMs they are waiting for.
__global__ void __launch_bounds__(128, 10) k_xfer(Ctrl c, int layer, XferArgs x, int mode) {
    const int n = c.plan_n[layer];
    const int E = c.E;
    const int total = n * XFER_CHUNKS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
        const int ci = w / XFER_CHUNKS, ch = w % XFER_CHUNKS;
        const int4 cmd = c.plan_cmd[layer * E + ci];
        const int e = cmd.x, dir = cmd.y, dst = cmd.z, src = cmd.w;
        if ((mode == 1 && dir != 0) || (mode == 2 && dir != 1) || (mode == 3 && dir != -1)) continue;
        if (dir == 1) {
            const uint4* s = reinterpret_cast<const uint4*>(x.hi_img[e]);
            uint4* d = reinterpret_cast<uint4*>(x.layer_base + x.hi_base + (i64)dst * x.hi.bytes);
            const i64 nvec = (x.hi.bits == 16 ? (i64)3 * x.I * x.H * 2 : x.hi.bytes) / 16;
            const i64 per = (nvec + XFER_CHUNKS - 1) / XFER_CHUNKS;
            const i64 v0 = ch * per, v1 = min(nvec, v0 + per);
            for (i64 v = v0 + threadIdx.x; v < v1; v += 4 * blockDim.x) {
                uint4 r[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) if (v + u * blockDim.x < v1) r[u] = s[v + u * blockDim.x];
#pragma unroll
                for (int u = 0; u < 4; ++u) if (v + u * blockDim.x < v1) d[v + u * blockDim.x] = r[u];
            }
        } else if (dir == 0) {
            if (mode != 1) continue;
            const uint4* s = reinterpret_cast<const uint4*>(x.layer_base + (i64)src * x.lo.bytes);
            uint4* d = reinterpret_cast<uint4*>(x.layer_base + (i64)dst * x.lo.bytes);
            const i64 nvec = x.lo.bytes / 16;
            const i64 per = (nvec + XFER_CHUNKS - 1) / XFER_CHUNKS;
            const i64 v0 = ch * per, v1 = min(nvec, v0 + per);
            for (i64 v = v0 + threadIdx.x; v < v1; v += blockDim.x) d[v] = s[v];
        } else {
            // demotion: quantise the 3 matrices of the HIGH block into the LOW block
            const uint8_t* hs = x.layer_base + x.hi_base + (i64)src * x.hi.bytes;
            uint8_t* ls = x.layer_base + (i64)dst * x.lo.bytes;
            const int g = x.g;
            const i64 gpr0 = x.H / g, gpr2 = x.I / g;                       // groups per row
            const i64 ngrp = (i64)2 * x.I * gpr0 + (i64)x.H * gpr2;
            const i64 per = (ngrp + XFER_CHUNKS - 1) / XFER_CHUNKS;
            const i64 g0 = ch * per, g1 = min(ngrp, g0 + per);
            for (i64 q = g0 + warp; q < g1; q += blockDim.x / 32) {
                int m; i64 row, gi, K;
                if (q < (i64)2 * x.I * gpr0) { m = (int)(q / (x.I * gpr0)); const i64 r = q % (x.I * gpr0); row = r / gpr0; gi = r % gpr0; K = x.H; }
                else { m = 2; const i64 r = q - (i64)2 * x.I * gpr0; row = r / gpr2; gi = r % gpr2; K = x.I; }
                const uint8_t* sc = hs + m * x.hi.codes_stride;
                const uint8_t* ssc = x.hi.bits == 16 ? nullptr : hs + x.hi.scales_off + m * x.hi.scales_stride;
                const uint8_t* sz = x.hi.bits == 16 ? nullptr : hs + x.hi.zeros_off + m * x.hi.zeros_stride;
                const i64 G = K / g;
                uint8_t* dc = ls + m * x.lo.codes_stride + row * (K * x.lo.bits / 8);
                __nv_bfloat16* dsc = reinterpret_cast<__nv_bfloat16*>(ls + x.lo.scales_off + m * x.lo.scales_stride) + row * G + gi;
                uint8_t* dz = ls + x.lo.zeros_off + m * x.lo.zeros_stride + row * G + gi;
                // slots hold codes in the pair-interleaved packing (dx_quant.cuh) on both sides
                if (g == 32)      { float wv[1]; dxq_fetch_group<1>(sc, x.hi.bits, ssc, sz, row, gi, K, g, lane, wv, true); dxq_quantize_group<1>(wv, x.lo.bits, gi, K, lane, dc, dsc, dz, true); }
                else if (g == 64) { float wv[2]; dxq_fetch_group<2>(sc, x.hi.bits, ssc, sz, row, gi, K, g, lane, wv, true); dxq_quantize_group<2>(wv, x.lo.bits, gi, K, lane, dc, dsc, dz, true); }
                else              { float wv[4]; dxq_fetch_group<4>(sc, x.hi.bits, ssc, sz, row, gi, K, g, lane, wv, true); dxq_quantize_group<4>(wv, x.lo.bits, gi, K, lane, dc, dsc, dz, true); }
            }
        }
    }
}

// ------------------------------------------------------------------ f-1: cross-layer correlation prefetch
// ("proactively prefetches experts predicted to become hot by leveraging cross-layer activation
// correlations"; SPEC.md:337-392 CorrelationModel / update_correlation / prefetch_candidates.)
// corr[e][e'] (pair of layers l, l+1) += 1 for every expert e layer l chose and e' layer l+1 chose for the same
// token: k*k increments per token (SPEC.md update_correlation).  Integer sums: order-free, bit-exact.
// idx_prev NULL: no update (the previous layer routed another batch); idx is also saved to idx_save for the next
// layer.  Programmatic dependent launch keeps it inside the forward's launch chain.
__global__ void k_corr(const int32_t* __restrict__ idx_prev, const int32_t* __restrict__ idx, int T, int k, int E,
                       uint32_t* __restrict__ corr, int32_t* __restrict__ idx_save) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < T * k) idx_save[i] = idx[i];
    if (!idx_prev || i >= T * k * k) return;
    const int t = i / (k * k), j = (i / k) % k, j2 = i % k;
    const int a = idx_prev[t * k + j], b = idx[t * k + j2];
    if (a >= 0 && a < E && b >= 0 && b < E) atomicAdd(&corr[(size_t)a * E + b], 1u);
}
// Prefetch candidates for layer `layer` (= l + 1) from layer l's current routing idx_cur [T][k]: score(e') =
// sum over the T*k chosen (t, j) of corr[idx_cur[t][j]][e'] (u64, exact); eligible e' are LOW-tier, not in flight,
// score > 0; up to f of them by (score desc, id asc), each paired with the next lowest free HIGH block in ascending
// order (the blocks the next plan's promotions take first).  out[i] = {expert, block}; *n_out = count.
__global__ void __launch_bounds__(512) k_prefetch(Ctrl c, int layer, const uint32_t* __restrict__ corr,
                                                  const int32_t* __restrict__ idx_cur, int T, int k, int f,
                                                  int4* __restrict__ out, int32_t* __restrict__ n_out) {
    __shared__ unsigned long long best[16];
    __shared__ int32_t freeb[64];
    __shared__ int32_t nfree;
    const int E = c.E, base = layer * E, ob = layer * (E + c.s);
    const int e = threadIdx.x;
    unsigned long long sc = 0;
    if (e < E) {
        for (int q = 0; q < T * k; ++q) {
            const int a = idx_cur[q];
            if (a >= 0 && a < E) sc += corr[(size_t)a * E + e];
        }
        if (c.tier[base + e] != 0 || c.pend_dir[base + e] != 0) sc = 0;
    }
    if (threadIdx.x == 0) {
        int nf = 0;
        const int cap = c.cap_hi[layer];
        for (int b = 0; b < cap && nf < 64; ++b)
            if (c.hi_owner[ob + b] < 0) freeb[nf++] = b;
        nfree = nf;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int n = 0;
    const int fmax = min(f, nfree);
    for (int r = 0; r < fmax; ++r) {
        // key: score in the high bits, (E - 1 - id) in the low 16 bits: max key = highest score, lowest id
        unsigned long long key = (sc > 0 && e < E) ? ((sc << 16) | (unsigned long long)(0xFFFF - e)) : 0ull;
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
            key = y > key ? y : key;
        }
        if (lane == 0) best[warp] = key;
        __syncthreads();
        unsigned long long m = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = best[w] > m ? best[w] : m;
        __syncthreads();
        if (m == 0) break;
        const int pick = 0xFFFF - (int)(m & 0xFFFF);
        if (e == pick) sc = 0;
        if (threadIdx.x == 0) out[n] = make_int4(pick, freeb[n], 0, 0);
        ++n;
    }
    if (threadIdx.x == 0) *n_out = n;
}

}  // namespace

void launch_fold(const Ctrl& c, int layer, u64 B_tot, cudaStream_t st) {
    dx_launch(k_fold, dim3(1), dim3(CTRL_THREADS), 0, st, g_dx_pdl, c, layer, B_tot, 1.0 - c.alpha);
}

void launch_plan(const Ctrl& c, int layer, int finalize, cudaStream_t st) {
    dx_launch(k_plan, dim3(1), dim3(CTRL_THREADS), 0, st, g_dx_pdl, c, layer, finalize);
}

void launch_corr(const int32_t* idx_prev, const int32_t* idx, int T, int k, int E, uint32_t* corr, int32_t* idx_save,
                 cudaStream_t st) {
    const int n = T * k * k;
    if (n <= 0) return;
    dx_launch(k_corr, dim3((n + 255) / 256), dim3(256), 0, st, g_dx_pdl, idx_prev, idx, T, k, E, corr, idx_save);
}

void launch_prefetch(const Ctrl& c, int layer, const uint32_t* corr, const int32_t* idx_cur, int T, int k, int f,
                     int4* out, int32_t* n_out, cudaStream_t st) {
    k_prefetch<<<1, 512, 0, st>>>(c, layer, corr, idx_cur, T, k, f, out, n_out);
}

void launch_manual(const Ctrl& c, int layer, const int2* cmds, int n, int32_t* status, cudaStream_t st) {
    k_manual<<<1, 32, 0, st>>>(c, layer, cmds, n, status);
}

void launch_transitions(const Ctrl& c, int layer, const XferArgs& x, int max_cmds, int mode,
                        cudaStream_t st) {
    int grid = max_cmds * XFER_CHUNKS;
    // finalize (modes 1, 2: synchronous on the compute stream, nothing to overlap) may take the whole GPU;
    // runtime transitions (mode 0, side stream) use at most one lean block per SM, which fits beside the
    // SM's persistent GEMM CTA, so the GEMMs keep every SM while the transfer runs
#ifndef DX_XFER_BLOCKS
#define DX_XFER_BLOCKS DX_NUM_SMS
#endif
    // demotions of runtime plans (mode 3; DX_DEMOTE_BLOCKS caps the grid): measured on C5 decode, 16 blocks took
    // 2.6 ms per plan and 4 blocks 10 ms (the warp-per-group quantiser is latency-bound), both past the publish
    // lag, while one lean block per SM (0.37 ms) exposed ~10 % -- so the default stays at one per SM
    static const int dem_blocks = [] { const char* e = getenv("DX_DEMOTE_BLOCKS"); return e ? atoi(e) : DX_NUM_SMS; }();
    const int cap = mode == 0 ? DX_XFER_BLOCKS : (mode == 3 ? dem_blocks : 4 * DX_NUM_SMS);
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    k_xfer<<<grid, 128, 0, st>>>(c, layer, x, mode);
}
