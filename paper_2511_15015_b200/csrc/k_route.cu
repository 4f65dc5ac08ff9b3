// k_route.cu -- router logits (a1), warp-shuffle top-k + softmax gates + hotness counters (a2, a3),
// stable permutation by expert (a4) and the weighted combine (a8).
//   Eq. 1: K = topk({g_i(x)}), y = sum_{j in K} g_j E_j(x).
//   "records the selected experts and accumulates gating probabilities".
// Readings: R-G1 (ties -> lower id, gates = softmax over the k selected logits), R-G2 (dx_expf),
// R-H1 (cnt u32, mass = sum rint(g * 2^24) u64: integer sums are order-free => bit-exact).
#include "dx_common.cuh"
#include <cstdio>

#define ROUTE_TOK_PER_BLK 8
#define ROUTE_MAX_E 512
#define ROUTE_MAX_K 16

namespace {

// ------------------------------------------------------------------ a1: logits = x Wr^T (+b), fp32
// Tensor-core router (mma.sync m16n8k16, bf16 products exact, fp32 accumulate): block = 8 experts x 16
// tokens, 16 warps each taking every 16th K step (short per-warp load chains, all fragment loads of a warp
// in flight at once; x is L2-resident).  The 16 warp partials are summed in smem in warp order, so the
// logits are deterministic.
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__global__ void __launch_bounds__(512) k_router(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wr,
                                                const float* __restrict__ bias, int T, int E, int H,
                                                float* __restrict__ logits) {
    __shared__ float red[16][16][9];                      // [warp][token][expert] partials
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int e0 = blockIdx.x * 8, t0 = blockIdx.y * 16;
    const int ta = t0 + g, tb = t0 + g + 8, e = e0 + g;
    const uint32_t* xa = reinterpret_cast<const uint32_t*>(x + (size_t)min(ta, T - 1) * H) + q;
    const uint32_t* xb = reinterpret_cast<const uint32_t*>(x + (size_t)min(tb, T - 1) * H) + q;
    const uint32_t* we = reinterpret_cast<const uint32_t*>(wr + (size_t)min(e, E - 1) * H) + q;
    const int nsteps = H / 16;
    float c[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    constexpr int U = 8;
    for (int s0 = warp; s0 < nsteps; s0 += 16 * U) {
        uint32_t f[U][6];
#pragma unroll
        for (int u = 0; u < U; ++u) {                      // all loads of the batch first
            const int s = s0 + 16 * u;
            if (s < nsteps) {
                const int k = s * 8;                       // 16 elements = 8 words per step
                f[u][0] = __ldg(xa + k); f[u][1] = __ldg(xb + k);
                f[u][2] = __ldg(xa + k + 4); f[u][3] = __ldg(xb + k + 4);
                f[u][4] = __ldg(we + k); f[u][5] = __ldg(we + k + 4);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (s0 + 16 * u < nsteps) mma16816(c, f[u][0], f[u][1], f[u][2], f[u][3], f[u][4], f[u][5]);
    }
    red[warp][g][2 * q] = c[0];
    red[warp][g][2 * q + 1] = c[1];
    red[warp][g + 8][2 * q] = c[2];
    red[warp][g + 8][2 * q + 1] = c[3];
    __syncthreads();
    if (threadIdx.x < 128) {
        const int tl = threadIdx.x >> 3, el = threadIdx.x & 7;   // 16 tokens x 8 experts
        const int t = t0 + tl, ee = e0 + el;
        if (t < T && ee < E) {
            float v = red[0][tl][el];
#pragma unroll
            for (int w = 1; w < 16; ++w) v += red[w][tl][el];
            logits[(size_t)t * E + ee] = bias ? v + bias[ee] : v;
        }
    }
}

__device__ __forceinline__ bool better(float a, int ea, float b, int eb) {
    return a > b || (a == b && ea < eb);
}

// Order-preserving u32 key of a float (larger float -> larger key); 0 = excluded (below every value).
__device__ __forceinline__ uint32_t fkey(float f) {
    uint32_t u = __float_as_uint(f);
    if (u == 0x80000000u) u = 0u;                          // -0 ties with +0 (float compare)
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
// k rounds of warp arg-max over E = 32 * NVT values (lane holds experts lane + 32 i): per round the best
// value by a max-reduction of order-preserving keys, ties to the lower expert id by a min-reduction
// (R-G1); sel_* in rank order.
template <int NVT>
__device__ __forceinline__ void topk_warp(const float (&v)[NVT], uint32_t taken, int k, int lane,
                                          float (&sel_v)[ROUTE_MAX_K], int (&sel_e)[ROUTE_MAX_K]) {
    uint32_t key[NVT];
#pragma unroll
    for (int i = 0; i < NVT; ++i) key[i] = ((taken >> i) & 1u) ? 0u : fkey(v[i]);
#pragma unroll
    for (int j = 0; j < ROUTE_MAX_K; ++j) {
        if (j >= k) break;
        uint32_t bk = 0u;
        int bi = 0;
#pragma unroll
        for (int i = 0; i < NVT; ++i)
            if (key[i] > bk) { bk = key[i]; bi = i; }          // ascending i: lowest expert on ties
        const uint32_t kmax = __reduce_max_sync(0xffffffffu, bk);
        const uint32_t mine = (bk == kmax && kmax != 0u) ? (uint32_t)(lane + 32 * bi) : 0xffffffffu;
        const uint32_t emin = __reduce_min_sync(0xffffffffu, mine);
        if (mine == emin) {
#pragma unroll
            for (int i = 0; i < NVT; ++i)
                if (i == bi) key[i] = 0u;
        }
        sel_v[j] = fkey_inv(kmax);
        sel_e[j] = (int)emin;
    }
}

// ------------------------------------------------------------------ a2 + a3: top-k, gates, counters
// One warp per token (8 tokens per block), k rounds of (value desc, id asc) warp arg-max over NVT
// logits per lane; per-block shared histograms merged into the layer's global accumulators with one
// atomic per touched expert.
template <typename Tv>
__device__ Tv block_excl_scan(Tv v, Tv* tmp, Tv* total);
__device__ void scan_tail(const int32_t* __restrict__ hist, int nblk, int E, int32_t* __restrict__ base,
                          int32_t* __restrict__ off, int32_t* __restrict__ act_e, int32_t* __restrict__ n_act,
                          const RouteStats& rs);

template <int NVT>
__global__ void __launch_bounds__(256) k_route(const float* __restrict__ logits, int T, int E, int k,
                                               int e_lo, int e_cnt, int32_t* __restrict__ idx_out,
                                               float* __restrict__ gate_out, int32_t* __restrict__ hist,
                                               uint32_t* __restrict__ cnt_acc, u64* __restrict__ mass_acc,
                                               int32_t* __restrict__ base, int32_t* __restrict__ off,
                                               int32_t* __restrict__ act_e, int32_t* __restrict__ n_act,
                                               RouteStats rs, unsigned* __restrict__ done) {
    __shared__ uint32_t cnt_s[ROUTE_MAX_E];
    __shared__ u64 mass_s[ROUTE_MAX_E];
    for (int e = threadIdx.x; e < E; e += blockDim.x) { cnt_s[e] = 0; mass_s[e] = 0; }
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * ROUTE_TOK_PER_BLK + warp;
    if (t < T) {
        float v[NVT];
        uint32_t taken = 0;
        const float* lrow = logits + (size_t)t * E;
#pragma unroll
        for (int i = 0; i < NVT; ++i) {
            const int e = lane + 32 * i;
            v[i] = e < E ? lrow[e] : -INFINITY;
            if (e >= E) taken |= 1u << i;
        }
        float sel_v[ROUTE_MAX_K];
        int sel_e[ROUTE_MAX_K];
        topk_warp<NVT>(v, taken, k, lane, sel_v, sel_e);
        // gates: softmax over the selected logits, sequential fp32 sum in rank order (R-G2)
        float ev[ROUTE_MAX_K];
        float sum = 0.0f;
#pragma unroll
        for (int j = 0; j < ROUTE_MAX_K; ++j) {
            if (j >= k) break;
            ev[j] = dx_expf(__fsub_rn(sel_v[j], sel_v[0]));
            sum = (j == 0) ? ev[0] : __fadd_rn(sum, ev[j]);
        }
        float my_ev = 0.0f;                             // lane j < k handles rank j (no divergent loop)
        int my_e = 0;
#pragma unroll
        for (int j = 0; j < ROUTE_MAX_K; ++j)
            if (j == lane) { my_ev = ev[j]; my_e = sel_e[j]; }
        if (lane < k) {
            const float gte = __fdiv_rn(my_ev, sum);
            idx_out[(size_t)t * k + lane] = my_e;
            gate_out[(size_t)t * k + lane] = gte;
            atomicAdd(&cnt_s[my_e], 1u);
            atomicAdd(&mass_s[my_e], (u64)rintf(__fmul_rn(gte, 16777216.0f)));
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        hist[(size_t)blockIdx.x * E + e] = (int32_t)cnt_s[e];
        const int le = e - e_lo;
        if (cnt_s[e] && le >= 0 && le < e_cnt && cnt_acc) {
            atomicAdd(&cnt_acc[le], cnt_s[e]);
            atomicAdd(&mass_acc[le], mass_s[e]);
        }
    }
    // the last block to finish runs the offset scan (a4) for the whole forward
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    scan_tail(hist, gridDim.x, E, base, off, act_e, n_act, rs);
    if (threadIdx.x == 0) *done = 0;
}

// ------------------------------------------------------------------ a2-a4 in ONE block (decode batches)
// T*k <= ROUTE1_MAX_ENT: top-k + gates + counters (as k_route), then the offsets scan, the active list and
// the stable placement (entry i's row = off[e] + #{i' < i : e_i' = e}) all in shared memory -- no
// cross-block completion counter, no second launch for the ranks.
#define ROUTE1_MAX_ENT 512
#define ROUTE1_CHUNKS 16
template <typename Tv>
__device__ Tv block_excl_scan(Tv v, Tv* tmp, Tv* total);
#ifdef DX_ROUTE_PROF
__device__ unsigned g_route1_calls = 0;
#define R1P(i) do { if (threadIdx.x == 0) tp[i] = clock64(); } while (0)
#else
#define R1P(i) do {} while (0)
#endif
template <int NVT>
__global__ void __launch_bounds__(512) k_route1(const float* __restrict__ logits, int T, int E, int k, int e_lo,
                                                int e_cnt, int32_t* __restrict__ idx_out, float* __restrict__ gate_out,
                                                uint32_t* __restrict__ cnt_acc, u64* __restrict__ mass_acc,
                                                int32_t* __restrict__ off, int32_t* __restrict__ act_e,
                                                int32_t* __restrict__ n_act, int32_t* __restrict__ perm,
                                                int32_t* __restrict__ inv, RouteStats rs) {
#ifdef DX_ROUTE_PROF
    long long tp[8] = {0};
#endif
    R1P(0);
    __shared__ int16_t ent_s[ROUTE1_MAX_ENT];                // expert of every entry (t*k + j)
    __shared__ uint32_t gm_s[ROUTE1_MAX_ENT];                // rint(gate * 2^24) of every entry (R-H1)
    __shared__ int32_t tmp[32];
    __shared__ int32_t total_s, na_s;
    extern __shared__ __align__(16) uint8_t dyn_s[];
    float* lg_s = reinterpret_cast<float*>(dyn_s);                              // [T][E] logits of the batch
    uint32_t* cmass = reinterpret_cast<uint32_t*>(lg_s + (size_t)T * E);        // [chunk][expert] mass
    int16_t* chist = reinterpret_cast<int16_t*>(cmass + ROUTE1_CHUNKS * E);     // [chunk][expert] counts, bases
    for (int i = threadIdx.x; i < ROUTE1_CHUNKS * E; i += blockDim.x) { chist[i] = 0; cmass[i] = 0; }
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    R1P(1);
    {
        const int n4 = T * E / 4;                            // E % 4 == 0 (route1_ok)
        const float4* src = reinterpret_cast<const float4*>(logits);
        float4* dst = reinterpret_cast<float4*>(lg_s);
#pragma unroll 4
        for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    R1P(2);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    // a2 + a3: one warp per token, k rounds of (value desc, id asc) warp arg-max, gates (R-G1, R-G2):
    // lane j < k evaluates e_j = dx_expf(l_j - l_0) for its rank, lane 0 forms the sequential rank-order
    // sum from shuffles (the same operations in the same order as one thread doing it all)
    for (int t = warp; t < T; t += nwarps) {
        float v[NVT];
        uint32_t taken = 0;
        const float* lrow = lg_s + (size_t)t * E;
#pragma unroll
        for (int i = 0; i < NVT; ++i) {
            const int e = lane + 32 * i;
            v[i] = e < E ? lrow[e] : -INFINITY;
            if (e >= E) taken |= 1u << i;
        }
        float sel_v[ROUTE_MAX_K];
        int sel_e[ROUTE_MAX_K];
        topk_warp<NVT>(v, taken, k, lane, sel_v, sel_e);
        float my_v = sel_v[0];
        int my_e = 0;
#pragma unroll
        for (int j = 0; j < ROUTE_MAX_K; ++j)
            if (j == lane) { my_v = sel_v[j]; my_e = sel_e[j]; }
        const float my_ev = lane < k ? dx_expf(__fsub_rn(my_v, sel_v[0])) : 0.0f;
        float part[ROUTE_MAX_K];
#pragma unroll
        for (int j = 0; j < ROUTE_MAX_K; ++j) part[j] = __shfl_sync(0xffffffffu, my_ev, j);
        float sum = part[0];
#pragma unroll
        for (int j = 1; j < ROUTE_MAX_K; ++j)
            if (j < k) sum = __fadd_rn(sum, part[j]);
        if (lane < k) {
            const float gte = __fdiv_rn(my_ev, sum);
            idx_out[(size_t)t * k + lane] = my_e;
            gate_out[(size_t)t * k + lane] = gte;
            ent_s[t * k + lane] = (int16_t)my_e;
            gm_s[t * k + lane] = (uint32_t)rintf(__fmul_rn(gte, 16777216.0f));
        }
    }
    __syncthreads();
    R1P(3);
    // per 32-entry chunk (one warp each): same-expert groups by match_any -> in-chunk rank, count, mass
    const int n = T * k;
    const int ci = warp, i = warp * 32 + lane;               // n <= 512 = 16 warps x 32 entries
    const bool have = i < n;
    const int ei = have ? ent_s[i] : -1 - lane;
    const unsigned same = __match_any_sync(0xffffffffu, ei);
    const int rk = __popc(same & ((1u << lane) - 1u));
    const uint32_t gsum = __reduce_add_sync(same, have ? gm_s[i] : 0u);
    if (have && rk == 0) {
        chist[ci * E + ei] = (int16_t)__popc(same);
        cmass[ci * E + ei] = gsum;
    }
    __syncthreads();
    // per expert (thread e): totals in chunk order (integer sums: order-free), offsets scan, active list,
    // hotness accumulators, chunk bases
    const int e = threadIdx.x;
    uint32_t c = 0;
    u64 m = 0;
    if (e < E) {
#pragma unroll
        for (int c2 = 0; c2 < ROUTE1_CHUNKS; ++c2) {
            c += (uint32_t)chist[c2 * E + e];
            m += cmass[c2 * E + e];
        }
        if (c) {
            const int le = e - e_lo;
            if (le >= 0 && le < e_cnt && cnt_acc) {
                atomicAdd(&cnt_acc[le], c);
                atomicAdd(&mass_acc[le], m);
            }
        }
    }
    R1P(4);
    const int32_t o = block_excl_scan<int32_t>((int32_t)c, tmp, &total_s);
    const int32_t a = block_excl_scan<int32_t>(c > 0 ? 1 : 0, tmp, &na_s);
    // active list HIGH tier first (the grouped GEMMs hand out work items in this order, heaviest first)
    __shared__ int32_t nhi_s;
    const int32_t hi = (e < E && c && rs.tier && rs.tier[e]) ? 1 : 0;
    const int32_t ah = block_excl_scan<int32_t>(hi, tmp, &nhi_s);
    if (e < E) {
        off[e] = o;
        if (c) act_e[hi ? ah : nhi_s + (a - ah)] = e;
        int run = o;
#pragma unroll
        for (int c2 = 0; c2 < ROUTE1_CHUNKS; ++c2) {
            const int b = chist[c2 * E + e];
            chist[c2 * E + e] = (int16_t)run;
            run += b;
        }
    }
    if (rs.stats && rs.tier) {                               // algorithmic weight bytes of this forward
        if (threadIdx.x == 0) {                               // (profiling): 3 atomics per forward
            const u64 nh = (u64)nhi_s, nl = (u64)na_s - nh;
            atomicAdd(&rs.stats[0], nh * rs.b10 + nl * rs.b00);
            atomicAdd(&rs.stats[1], nh * rs.b11 + nl * rs.b01);
            atomicAdd(&rs.stats[2], (u64)na_s);
        }
    }
    if (threadIdx.x == 0) { off[E] = total_s; *n_act = na_s; }
    __syncthreads();
    R1P(5);
    // a4: stable placement (entry order t asc, j asc): pos = off[e] + earlier chunks + in-chunk rank
    if (have) {
        const int pos = chist[ci * E + ei] + rk;
        perm[pos] = i;
        inv[i] = pos;
    }
#ifdef DX_ROUTE_PROF
    R1P(6);
    if (threadIdx.x == 0) {
        const unsigned c = atomicAdd(&g_route1_calls, 1u);
        if (c == 300)
            printf("route1 T=%d clocks: wait %lld copy %lld topk %lld chunks %lld scans %lld place %lld total %lld\n", T,
                   tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4], tp[6] - tp[5], tp[6] - tp[0]);
    }
#endif
}

// x rows gathered into the permuted order (B operand of the gate/up GEMM): Xp[inv[i]] = x[i / k]; one
// warp per entry, 16 B per lane per step
__global__ void __launch_bounds__(256) k_gather(const int32_t* __restrict__ inv, int n, int k, const __nv_bfloat16* __restrict__ x,
                                                int H, __nv_bfloat16* __restrict__ Xp) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= n) return;
    const int pos = inv[i];
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)(i / k) * H);
    uint4* dst = reinterpret_cast<uint4*>(Xp + (size_t)pos * H);
    for (int h = lane; h < H / 8; h += 32) dst[h] = src[h];
}

// ------------------------------------------------------------------ a4: offsets + stable scatter
template <typename Tv>
__device__ Tv block_excl_scan(Tv v, Tv* tmp /*[32]*/, Tv* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    Tv x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        Tv y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) tmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        Tv s = lane < nw ? tmp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            Tv y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) tmp[lane] = s;
    }
    __syncthreads();
    const Tv before = (warp > 0 ? tmp[warp - 1] : 0) + x - v;
    if (total) *total = tmp[nw - 1];
    __syncthreads();
    return before;
}

// Offsets of every expert's row segment, per-route-block bases and the active-expert list.  Run by
// the LAST route block to finish (threadfence + completion counter), so routing and its scan are one
// launch.  256 threads, 2 experts per thread (E <= 512).
__device__ void scan_tail(const int32_t* __restrict__ hist, int nblk, int E, int32_t* __restrict__ base,
                          int32_t* __restrict__ off, int32_t* __restrict__ act_e, int32_t* __restrict__ n_act,
                          const RouteStats& rs) {
    __shared__ int32_t tmp[32];
    __shared__ int32_t total_s, na_s;
    const int e0 = 2 * threadIdx.x, e1 = e0 + 1;
    int32_t t0 = 0, t1 = 0;
    for (int b = 0; b < nblk; ++b) {
        if (e0 < E) t0 += __ldcg(hist + (size_t)b * E + e0);
        if (e1 < E) t1 += __ldcg(hist + (size_t)b * E + e1);
    }
    const int32_t o = block_excl_scan<int32_t>(t0 + t1, tmp, &total_s);
    const int32_t a = block_excl_scan<int32_t>((t0 > 0) + (t1 > 0), tmp, &na_s);
    // active list HIGH tier first (the grouped GEMMs hand out work items in this order, heaviest first)
    __shared__ int32_t nhi_s;
    const bool h0 = e0 < E && t0 > 0 && rs.tier && rs.tier[e0], h1 = e1 < E && t1 > 0 && rs.tier && rs.tier[e1];
    const int32_t ah = block_excl_scan<int32_t>((int32_t)h0 + (int32_t)h1, tmp, &nhi_s);
    int32_t ahi = ah, alo = nhi_s + (a - ah);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int e = h ? e1 : e0;
        const int32_t tot = h ? t1 : t0;
        if (e >= E) continue;
        const int32_t oe = h ? o + t0 : o;
        off[e] = oe;
        if (tot > 0) act_e[(h ? h1 : h0) ? ahi++ : alo++] = e;
        int32_t run = oe;
        for (int b = 0; b < nblk; ++b) {
            base[(size_t)b * E + e] = run;
            run += __ldcg(hist + (size_t)b * E + e);
        }
    }
    if (rs.stats && rs.tier) {                  // algorithmic weight bytes of this forward (profiling)
        if (threadIdx.x == 0) {
            const u64 nh = (u64)nhi_s, nl = (u64)na_s - nh;
            atomicAdd(&rs.stats[0], nh * rs.b10 + nl * rs.b00);
            atomicAdd(&rs.stats[1], nh * rs.b11 + nl * rs.b01);
            atomicAdd(&rs.stats[2], (u64)na_s);
        }
    }
    if (threadIdx.x == 0) { off[E] = total_s; *n_act = na_s; }
}

// One block per entry (t*k + j): its row position = base[block][e] + number of earlier entries of the
// same expert inside its route block (the stable counting-sort order: t asc, j asc); the block then
// copies x[t] into Xp[pos] (the B operand of the gate/up GEMM) when Xp != NULL.
__global__ void __launch_bounds__(128) k_place(const int32_t* __restrict__ idx, int T, int E, int k,
                                               const int32_t* __restrict__ base, int32_t* __restrict__ perm,
                                               int32_t* __restrict__ inv, const __nv_bfloat16* __restrict__ x,
                                               int H, __nv_bfloat16* __restrict__ Xp) {
    __shared__ int pos_s;
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int i = blockIdx.x;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int b = (i / k) / ROUTE_TOK_PER_BLK;
        const int e = idx[i];
        int r = 0;
        for (int q = b * ROUTE_TOK_PER_BLK * k + lane; q < i; q += 32) r += (idx[q] == e);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        if (lane == 0) {
            const int pos = base[(size_t)b * E + e] + r;
            perm[pos] = i;
            inv[i] = pos;
            pos_s = pos;
        }
    }
    if (!Xp) return;
    __syncthreads();
    const int pos = pos_s;
    const __nv_bfloat16* src = x + (size_t)(i / k) * H;
    for (int h = threadIdx.x * 8; h < H; h += blockDim.x * 8)
        *reinterpret_cast<uint4*>(Xp + (size_t)pos * H + h) = *reinterpret_cast<const uint4*>(src + h);
}

// ------------------------------------------------------------------ a8: y_t = bf16(sum_j Y[t,j])
// inv == NULL: Y rows in entry order (t*k + j); else Y rows in permuted order, entry i at row inv[i]
// (expert-parallel combine: the rows come back from their owners in dispatch order).
__global__ void k_combine(const __nv_bfloat16* __restrict__ Y, int k, int H, __nv_bfloat16* __restrict__ y,
                          const int32_t* __restrict__ inv) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int t = blockIdx.x;
    for (int h = threadIdx.x * 8; h < H; h += blockDim.x * 8) {
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
        for (int j = 0; j < k; ++j) {
            const size_t row = inv ? (size_t)inv[(size_t)t * k + j] : (size_t)t * k + j;
            uint4 v = *reinterpret_cast<const uint4*>(Y + row * H + h);
            const uint16_t* b = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], dx_bf2f(b[i]));
        }
        __align__(16) __nv_bfloat16 o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16_rn(acc[i]);
        *reinterpret_cast<uint4*>(y + (size_t)t * H + h) = *reinterpret_cast<const uint4*>(o);
    }
}

// ------------------------------------------------------------------ expert parallelism (a15)
// Owner side: rows arrive with (local expert, gate); k = 1 routing is given.  Per block of 8 rows:
// copy idx/gate into the workspace, shared histograms, hotness counters (owner-side counting, SURVEY
// §8(e)), then the last block runs the offset scan exactly as after top-k.
__global__ void __launch_bounds__(256) k_route_given(const int2* __restrict__ meta, int R, int E,
                                                     int32_t* __restrict__ idx_out, float* __restrict__ gate_out,
                                                     int32_t* __restrict__ hist, uint32_t* __restrict__ cnt_acc,
                                                     u64* __restrict__ mass_acc, int32_t* __restrict__ base,
                                                     int32_t* __restrict__ off, int32_t* __restrict__ act_e,
                                                     int32_t* __restrict__ n_act, RouteStats rs,
                                                     unsigned* __restrict__ done, int32_t* __restrict__ err) {
    __shared__ uint32_t cnt_s[ROUTE_MAX_E];
    __shared__ u64 mass_s[ROUTE_MAX_E];
    for (int e = threadIdx.x; e < E; e += blockDim.x) { cnt_s[e] = 0; mass_s[e] = 0; }
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    __syncthreads();
    const int r = blockIdx.x * ROUTE_TOK_PER_BLK + threadIdx.x;
    if (threadIdx.x < ROUTE_TOK_PER_BLK && r < R) {
        const int2 m = meta[r];
        const float g = __int_as_float(m.y);
        if (m.x < 0 || m.x >= E) {
            atomicExch(err, 2);
        } else {
            idx_out[r] = m.x;
            gate_out[r] = g;
            atomicAdd(&cnt_s[m.x], 1u);
            atomicAdd(&mass_s[m.x], (u64)rintf(__fmul_rn(g, 16777216.0f)));
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        hist[(size_t)blockIdx.x * E + e] = (int32_t)cnt_s[e];
        if (cnt_s[e] && cnt_acc) {
            atomicAdd(&cnt_acc[e], cnt_s[e]);
            atomicAdd(&mass_acc[e], mass_s[e]);
        }
    }
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    scan_tail(hist, gridDim.x, E, base, off, act_e, n_act, rs);
    if (threadIdx.x == 0) *done = 0;
}

// Source side after placement: metadata of every dispatched row (local expert id at its owner, gate
// bits) and per-owner row counts (rows for owner o are contiguous because experts are partitioned
// contiguously: [off[o*E_loc], off[(o+1)*E_loc]) ).
__global__ void k_ep_meta(const int32_t* __restrict__ perm, const int32_t* __restrict__ idx,
                          const float* __restrict__ gate, const int32_t* __restrict__ off, int n, int E_loc, int G,
                          int2* __restrict__ meta, int32_t* __restrict__ counts) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos < n) {
        const int ent = perm[pos];
        const int e = idx[ent];
        meta[pos] = make_int2(e % E_loc, __float_as_int(gate[ent]));
    }
    if (pos < G) counts[pos] = off[(pos + 1) * E_loc] - off[pos * E_loc];
}

// ------------------------------------------------------------------ trace-mode counters
__global__ void k_counts_from(const int32_t* __restrict__ idx, const float* __restrict__ gate, int T,
                              int E, int k, int e_lo, int e_cnt, uint32_t* __restrict__ cnt_acc,
                              u64* __restrict__ mass_acc, int32_t* __restrict__ err) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    for (int j = 0; j < k; ++j) {
        const int e = idx[(size_t)t * k + j];
        if (e < 0 || e >= E) { atomicExch(err, 2); continue; }
        for (int j2 = 0; j2 < j; ++j2)
            if (idx[(size_t)t * k + j2] == e) atomicExch(err, 1);
        const int le = e - e_lo;
        if (le < 0 || le >= e_cnt) continue;
        atomicAdd(&cnt_acc[le], 1u);
        atomicAdd(&mass_acc[le], (u64)rintf(__fmul_rn(gate[(size_t)t * k + j], 16777216.0f)));
    }
}

}  // namespace

int route_blocks(int T) { return (T + ROUTE_TOK_PER_BLK - 1) / ROUTE_TOK_PER_BLK; }

void launch_router(const __nv_bfloat16* x, const __nv_bfloat16* wr, const float* bias, int T, int E, int H,
                   float* logits, cudaStream_t st) {
    if (T <= 0) return;
    dim3 grid((E + 7) / 8, (T + 15) / 16);
    dx_launch(k_router, grid, dim3(512), 0, st, g_dx_pdl, x, wr, bias, T, E, H, logits);
}

void launch_route(const float* logits, int T, int E, int k, int e_lo, const RouteWs& ws,
                  uint32_t* cnt_acc, u64* mass_acc, const int32_t* tier, const u64 (&bytes)[2][2], cudaStream_t st) {
    if (T <= 0) return;
    const int nb = route_blocks(T), ec = cnt_acc ? E : 0;
    RouteStats rs{tier, bytes[0][0], bytes[0][1], bytes[1][0], bytes[1][1], ws.stats};
#define DX_ROUTE_ARGS logits, T, E, k, e_lo, ec, ws.idx, ws.gate, ws.hist, cnt_acc, mass_acc, ws.base, ws.off, \
                      ws.act_e, ws.n_act, rs, ws.done
    if (E <= 128)      dx_launch(k_route<4>, dim3(nb), dim3(256), 0, st, g_dx_pdl, DX_ROUTE_ARGS);
    else if (E <= 256) dx_launch(k_route<8>, dim3(nb), dim3(256), 0, st, g_dx_pdl, DX_ROUTE_ARGS);
    else               dx_launch(k_route<16>, dim3(nb), dim3(256), 0, st, g_dx_pdl, DX_ROUTE_ARGS);
#undef DX_ROUTE_ARGS
}

bool route1_ok(int T, int E, int k) { return T * k <= ROUTE1_MAX_ENT && E <= 512 && E % 4 == 0 && T * E <= 32768; }

void launch_route1(const float* logits, int T, int E, int k, int e_lo, const RouteWs& ws,
                   uint32_t* cnt_acc, u64* mass_acc, const int32_t* tier, const u64 (&bytes)[2][2], cudaStream_t st) {
    if (T <= 0) return;
    const int ec = cnt_acc ? E : 0;
    RouteStats rs{tier, bytes[0][0], bytes[0][1], bytes[1][0], bytes[1][1], ws.stats};
#define DX_R1_ARGS logits, T, E, k, e_lo, ec, ws.idx, ws.gate, cnt_acc, mass_acc, ws.off, ws.act_e, ws.n_act, \
                   ws.perm, ws.inv, rs
    static bool attr = false;
    if (!attr) {
        const int mx = 32768 * 4 + ROUTE1_CHUNKS * ROUTE_MAX_E * 6;
        cudaFuncSetAttribute(k_route1<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route1<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route1<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        attr = true;
    }
    const size_t sm = (size_t)T * E * 4 + (size_t)ROUTE1_CHUNKS * E * 6;
    if (E <= 128)      dx_launch(k_route1<4>, dim3(1), dim3(512), sm, st, g_dx_pdl, DX_R1_ARGS);
    else if (E <= 256) dx_launch(k_route1<8>, dim3(1), dim3(512), sm, st, g_dx_pdl, DX_R1_ARGS);
    else               dx_launch(k_route1<16>, dim3(1), dim3(512), sm, st, g_dx_pdl, DX_R1_ARGS);
#undef DX_R1_ARGS
}

void launch_gather(int T, int k, const RouteWs& ws, const __nv_bfloat16* x, int H, __nv_bfloat16* Xp, cudaStream_t st) {
    const int n = T * k;
    if (n <= 0 || !Xp) return;
    dx_launch(k_gather, dim3((n + 7) / 8), dim3(256), 0, st, g_dx_pdl, (const int32_t*)ws.inv, n, k, x, H, Xp);
}

void launch_place(int T, int E, int k, const RouteWs& ws, const __nv_bfloat16* x, int H, __nv_bfloat16* Xp,
                  cudaStream_t st) {
    if (T <= 0) return;
    dx_launch(k_place, dim3(T * k), dim3(128), 0, st, g_dx_pdl, (const int32_t*)ws.idx, T, E, k,
              (const int32_t*)ws.base, ws.perm, ws.inv, x, H, Xp);
}

void launch_combine(const __nv_bfloat16* Y, int T, int k, int H, __nv_bfloat16* y, cudaStream_t st,
                    const int32_t* inv) {
    if (T <= 0) return;
    int threads = H / 8 < 256 ? H / 8 : 256;
    dx_launch(k_combine, dim3(T), dim3(threads), 0, st, g_dx_pdl, Y, k, H, y, inv);
}

void launch_route_given(const int2* meta, int R, int E, const RouteWs& ws, uint32_t* cnt_acc, u64* mass_acc,
                        const int32_t* tier, const u64 (&bytes)[2][2], int32_t* err, cudaStream_t st) {
    if (R <= 0) return;
    RouteStats rs{tier, bytes[0][0], bytes[0][1], bytes[1][0], bytes[1][1], ws.stats};
    dx_launch(k_route_given, dim3(route_blocks(R)), dim3(256), 0, st, g_dx_pdl, meta, R, E, ws.idx, ws.gate, ws.hist,
              cnt_acc, mass_acc, ws.base, ws.off, ws.act_e, ws.n_act, rs, ws.done, err);
}

void launch_ep_meta(const RouteWs& ws, int n, int E_loc, int G, int2* meta, int32_t* counts, cudaStream_t st) {
    const int thr = 256, nb = ((n > G ? n : G) + thr - 1) / thr;
    dx_launch(k_ep_meta, dim3(nb > 0 ? nb : 1), dim3(thr), 0, st, g_dx_pdl, (const int32_t*)ws.perm,
              (const int32_t*)ws.idx, (const float*)ws.gate, (const int32_t*)ws.off, n, E_loc, G, meta, counts);
}

void launch_counts_from(const int32_t* idx, const float* gate, int T, int E, int k, int e_lo,
                        uint32_t* cnt_acc, u64* mass_acc, int32_t* err, cudaStream_t st) {
    if (T <= 0) return;
    k_counts_from<<<(T + 127) / 128, 128, 0, st>>>(idx, gate, T, E, k, e_lo, E, cnt_acc, mass_acc, err);
}
