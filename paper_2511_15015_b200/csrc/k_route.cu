// k_route.cu -- router logits (a1), warp-shuffle top-k + softmax gates + hotness counters (a2, a3),
// stable permutation by expert (a4) and the weighted combine (a8).
//   Eq. 1: K = topk({g_i(x)}), y = sum_{j in K} g_j E_j(x).
//   "records the selected experts and accumulates gating probabilities".
// Readings: R-G1 (ties -> lower id, gates = softmax over the k selected logits), R-G2 (dx_expf),
// R-H1 (cnt u32, mass = sum rint(g * 2^24) u64: integer sums are order-free => bit-exact).
#include "dx_common.cuh"
#include "dx_sm100.cuh"
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

// Router for larger T (prefill): a tiled tensor-core GEMM logits[T][E] = x[T][H] W_r[E][H]^T (+ b).  Block tile
// 32 tokens x 128 experts (T = 4096: 128 CTAs; 64-token tiles left 84 SMs idle: 34.8 -> 27.3 us), K in chunks of 64
// staged through shared memory by cp.async (double-buffered; 16-byte units XOR-swizzled by row so the ldmatrix row
// groups hit distinct banks), 8 warps of 16 tokens x 32 experts (1 x 4 mma.sync m16n8k16 tiles, fragments by
// ldmatrix).  Each logit is one warp's fp32 accumulation in K order: deterministic.  x is read once, W_r once per
// token tile (from L2).
constexpr int RT_M = 32, RT_N = 128, RT_K = 64, RT_LD = RT_K;   // rows of 8 16-byte units, unit c at c ^ (row & 7)
constexpr int RT_MI = RT_M / 32;               // 16-row m tiles per warp (8 warps: 2 along tokens x 4 along experts)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(pred ? 16 : 0));
}
__global__ void __launch_bounds__(256) k_router_tiled(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wr,
                                                      const float* __restrict__ bias, int T, int E, int H,
                                                      float* __restrict__ logits) {
    __shared__ __align__(16) __nv_bfloat16 xs[2][RT_M][RT_LD];
    __shared__ __align__(16) __nv_bfloat16 ws[2][RT_N][RT_LD];
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t0 = blockIdx.x * RT_M, e0 = blockIdx.y * RT_N;
    const int wm = (warp & 1) * (RT_M / 2), wn = (warp >> 1) * 32;   // warp tile origin in the block tile
    auto stage = [&](int buf, int k0) {
        // x: RT_M rows x 8 16-byte units; W_r: 128 rows x 8 units, over 256 threads
        for (int u = tid; u < (RT_M + RT_N) * 8; u += 256) {
            const int row = u >> 3, c = u & 7;
            if (row < RT_M) {
                const int t = t0 + row;
                cp_async16((uint32_t)__cvta_generic_to_shared(&xs[buf][row][(c ^ (row & 7)) * 8]),
                           x + (size_t)min(t, T - 1) * H + k0 + c * 8, t < T);
            } else {
                const int e = e0 + row - RT_M;
                const int wrow = row - RT_M;
                cp_async16((uint32_t)__cvta_generic_to_shared(&ws[buf][wrow][(c ^ (wrow & 7)) * 8]),
                           wr + (size_t)min(e, E - 1) * H + k0 + c * 8, e < E);
            }
        }
        asm volatile("cp.async.commit_group;");
    };
    float acc[RT_MI][4][4];
#pragma unroll
    for (int i = 0; i < RT_MI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0f;
    const int nk = H / RT_K;
    stage(0, 0);
    for (int kc = 0; kc < nk; ++kc) {
        const int buf = kc & 1;
        if (kc + 1 < nk) {
            stage(buf ^ 1, (kc + 1) * RT_K);
            asm volatile("cp.async.wait_group 1;");
        } else {
            asm volatile("cp.async.wait_group 0;");
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < RT_K; ks += 16) {
            uint32_t a[RT_MI][4], b[4][2];
#pragma unroll
            for (int i = 0; i < RT_MI; ++i) {               // A 16x16: rows wm+16i.., ldmatrix.x4
                const int r = wm + 16 * i + (lane & 15), cu = (ks >> 3) + (lane >> 4);
                const uint32_t ad = (uint32_t)__cvta_generic_to_shared(&xs[buf][r][(cu ^ (r & 7)) * 8]);
                asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                             : "=r"(a[i][0]), "=r"(a[i][1]), "=r"(a[i][2]), "=r"(a[i][3]) : "r"(ad));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {                   // B 16x8 from W_r rows (K contiguous), ldmatrix.x2
                const int r = wn + 8 * j + (lane & 7), cu = (ks >> 3) + ((lane >> 3) & 1);
                const uint32_t ad = (uint32_t)__cvta_generic_to_shared(&ws[buf][r][(cu ^ (r & 7)) * 8]);
                asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(b[j][0]), "=r"(b[j][1]) : "r"(ad));
            }
#pragma unroll
            for (int i = 0; i < RT_MI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) mma16816(acc[i][j], a[i][0], a[i][1], a[i][2], a[i][3], b[j][0], b[j][1]);
        }
        __syncthreads();
    }
    const int g = lane >> 2, q = lane & 3;
#pragma unroll
    for (int i = 0; i < RT_MI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = t0 + wm + 16 * i + g + 8 * h;
                const int e = e0 + wn + 8 * j + 2 * q;
                if (t < T) {
                    if (e < E) logits[(size_t)t * E + e] = bias ? acc[i][j][2 * h] + bias[e] : acc[i][j][2 * h];
                    if (e + 1 < E) logits[(size_t)t * E + e + 1] = bias ? acc[i][j][2 * h + 1] + bias[e + 1] : acc[i][j][2 * h + 1];
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
        hist[(size_t)e * gridDim.x + blockIdx.x] = (int32_t)cnt_s[e];     // [expert][route block]
        const int le = e - e_lo;
        if (cnt_s[e] && le >= 0 && le < e_cnt && cnt_acc) {
            atomicAdd(&cnt_acc[le], cnt_s[e]);
            atomicAdd(&mass_acc[le], mass_s[e]);
        }
    }
}

// ------------------------------------------------------------------ a1-a4 in ONE launch (decode batches)
// T*k <= RDEC_MAX_ENT entries.  The grid is ceil(T/16) clusters of CS CTAs x 512 threads (CS = 8 for H = 2048;
// every CTA is resident: the grid is far below the SM count and the next kernel is released with
// griddepcontrol.launch_dependents only after the grid barrier):
//   A (router mode) cluster c owns tokens [16c, 16c+16); CTA rank r computes partial logits over the K slice
//     [r H/CS, (r+1) H/CS) for all E experts (mma.sync m16n8k16: exact bf16 products, fp32 accumulation in K
//     order) into its shared memory;
//   B after a cluster barrier, CTA r takes tokens r, r + CS, ... of the tile (one warp per token): logit = the
//     CS partials read over distributed shared memory and summed in rank order (+ b), written to the logits
//     buffer; top-k + gates (R-G1, R-G2) to idx/gate and the per-entry exchange; the hotness counters take
//     integer atomics per entry (u32 cnt, u64 mass: order-free, R-H1);
//   one grid barrier (all entries routed), then
//   C every CTA recomputes the per-chunk expert histograms of all entries (match_any), the offsets scan and the
//     chunk bases in shared memory (identical in every CTA), CTA 0 publishes off / active list, and each CTA
//     places and gathers its share of the entries (perm / inv, Xp[pos] = x[t]) -- the stable order
//     (t asc, j asc) of a4.
// The router logits are deterministic (fixed slice partition and summation order per H).
#define RDEC_MAX_ENT 512
#define RDEC_CHUNKS (RDEC_MAX_ENT / 32)
template <typename Tv>
__device__ Tv block_excl_scan(Tv v, Tv* tmp, Tv* total);

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel_gpu(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// Grid-wide barrier over a {arrivals, generation} pair that resets itself (reusable across launches): read the
// generation, arrive (acq_rel), the last arrival resets the count and releases the next generation; the others
// poll the generation with acquire loads (no sleep: the wait is one L2 round trip after the last arrival).
__device__ __forceinline__ void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire_gpu(bar + 1);
        if (atom_add_acqrel_gpu(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            st_release_gpu(bar + 1, g + 1u);
        } else {
            const long long t0 = clock64();
            while (ld_acquire_gpu(bar + 1) == g)
                if (clock64() - t0 > 4000000000ll) __trap();   // ~2 s: a protocol bug, fail the launch
        }
    }
    __syncthreads();
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t local_addr, uint32_t rank) {
    uint32_t ra;
    float v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(rank));
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra));
    return v;
}

struct RouteDecArgs {
    const __nv_bfloat16* x;
    const __nv_bfloat16* wr;      // router mode (else logits_in)
    const float* bias;
    const float* logits_in;
    int T, E, k, H, e_lo, e_cnt, cs, ech;
    RouteWs ws;
    uint32_t* cnt_acc;
    u64* mass_acc;
    RouteStats rs;
    __nv_bfloat16* Xp;
};

#ifdef DX_RDEC_PROF
__device__ unsigned g_rdec_n = 0;
#define RDEC_T(i) if (threadIdx.x == 0) tstamp[i] = globaltimer_ns_r();
__device__ __forceinline__ unsigned long long globaltimer_ns_r() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#else
#define RDEC_T(i)
#endif
template <int NVT>
__global__ void __launch_bounds__(512) k_route_dec(const RouteDecArgs a) {
#ifdef DX_RDEC_PROF
    __shared__ unsigned long long tstamp[12];
#endif
    RDEC_T(0)
    extern __shared__ __align__(16) uint8_t dyn_s[];
    __shared__ int16_t ent_s[RDEC_MAX_ENT];
    __shared__ int16_t rk_s[RDEC_MAX_ENT];
    __shared__ int32_t tmp[32];
    __shared__ int32_t total_s, na_s, nhi_s;
    __shared__ __align__(8) uint64_t abar;
    __shared__ float bias_s[ROUTE_MAX_E];
    float* part = reinterpret_cast<float*>(dyn_s);                              // A/B: [16][E] partial logits
    int16_t* chist = reinterpret_cast<int16_t*>(dyn_s);                         // C: [chunk][E] counts -> bases
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int T = a.T, E = a.E, k = a.k, H = a.H, CS = a.cs;
    const uint32_t rank = CS > 1 ? cluster_rank() : 0u;
    const int t0 = (blockIdx.x / CS) * 16;                                      // this cluster's token tile
    // Router mode: the W_r slice of the first expert round (and the bias) are constant inputs, so their bulk copies
    // are issued before griddepcontrol.wait and overlap the previous kernel's tail; the x rows follow the wait.
    const int Hs = H / CS, pitch = Hs + 8;
    __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(dyn_s + (size_t)16 * E * 4);   // [16][pitch]
    __nv_bfloat16* wsm = xs + 16 * pitch;                                               // [ECH][pitch]
    const int ECH = a.ech;
    if (a.wr) {
        if (threadIdx.x == 0) {
            sm100::mbar_init(&abar, 1);
            sm100::fence_mbar_init();
            sm100::mbar_arrive_expect_tx(&abar, (uint32_t)((16 + min(ECH, E)) * Hs * 2));
        }
        __syncthreads();
        for (int r = threadIdx.x; r < min(ECH, E); r += blockDim.x)
            sm100::bulk_load(wsm + r * pitch, a.wr + (size_t)r * H + (size_t)rank * Hs, (uint32_t)(Hs * 2), &abar);
        if (a.bias && threadIdx.x < E) bias_s[threadIdx.x] = __ldg(a.bias + threadIdx.x);
    }
    DX_GRID_WAIT();
    RDEC_T(1)
    // this thread's expert's published tier (phase C's HIGH-first active list): read now, used after the barrier
    const int tier_e = ((int)threadIdx.x < E && a.rs.tier) ? __ldcg(a.rs.tier + threadIdx.x) : 0;
    if (a.wr) {
        // ---------------- A: partial router logits over this CTA's K slice (router in full precision).
        // The slice of the tile's 16 x rows and of W_r (ECH experts per round) is staged in shared memory by bulk
        // copies (one per row, rows padded by 16 B so the ldmatrix row groups hit distinct banks), then warp w
        // takes expert tiles w, w + 16, ... (mma.sync m16n8k16, fp32 accumulation in K order).
        uint32_t aph = 0;
        for (int e0 = 0; e0 < E; e0 += ECH) {
            const int ne = min(ECH, E - e0);
            if (e0 > 0) {                                     // later rounds: W_r and x after the previous compute
                if (threadIdx.x == 0) sm100::mbar_arrive_expect_tx(&abar, (uint32_t)((16 + ne) * Hs * 2));
                __syncthreads();
            }
            for (int r = e0 > 0 ? threadIdx.x : threadIdx.x + ne; r < 16 + ne; r += blockDim.x) {
                // round 0: only the 16 x rows (r = ne .. ne + 15); later rounds: x rows r < 16, then W rows
                const int rr = e0 > 0 ? r : r - ne;
                const __nv_bfloat16* src = rr < 16 ? a.x + (size_t)min(t0 + rr, T - 1) * H + (size_t)rank * Hs
                                                   : a.wr + (size_t)(e0 + rr - 16) * H + (size_t)rank * Hs;
                __nv_bfloat16* dst = rr < 16 ? xs + rr * pitch : wsm + (rr - 16) * pitch;
                sm100::bulk_load(dst, src, (uint32_t)(Hs * 2), &abar);
            }
            sm100::mbar_wait(&abar, aph);
            aph ^= 1u;
            const int g = lane >> 2, q = lane & 3;
            for (int et = warp; et < ne / 8; et += 16) {
                float c[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                const uint32_t xa = (uint32_t)__cvta_generic_to_shared(xs + (lane & 15) * pitch + 8 * (lane >> 4));
                const uint32_t wa = (uint32_t)__cvta_generic_to_shared(wsm + (et * 8 + (lane & 7)) * pitch + 8 * ((lane >> 3) & 1));
                for (int ks = 0; ks < Hs; ks += 16) {
                    uint32_t a0, a1, a2, a3, b0, b1;
                    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(xa + 2 * ks));
                    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(b0), "=r"(b1) : "r"(wa + 2 * ks));
                    mma16816(c, a0, a1, a2, a3, b0, b1);
                }
                const int ee = e0 + et * 8 + 2 * q;
                part[g * E + ee] = c[0];
                part[g * E + ee + 1] = c[1];
                part[(g + 8) * E + ee] = c[2];
                part[(g + 8) * E + ee + 1] = c[3];
            }
            __syncthreads();                                  // staging buffers free for the next round
        }
        if (CS > 1) cluster_barrier();
    }
    RDEC_T(2)
    // ---------------- B: logits (rank-ordered sum of the cluster's partials) + top-k + gates, one warp per token
    if (warp < 16 / CS) {
        const int tl = (int)rank + CS * warp;
        const int t = t0 + tl;
        if (t < T) {
            float v[NVT];
            uint32_t taken = 0;
            const uint32_t prow = (uint32_t)__cvta_generic_to_shared(part + tl * E);
#pragma unroll
            for (int i = 0; i < NVT; ++i) {
                const int e = lane + 32 * i;
                if (e >= E) {
                    v[i] = -INFINITY;
                    taken |= 1u << i;
                } else if (a.wr) {
                    float pv[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r)                 // every remote load in flight, then the ordered sum
                        if (r < CS) pv[r] = CS > 1 ? ld_cluster_f32(prow + 4 * e, r) : part[tl * E + e];
                    float sum = 0.0f;
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (r < CS) sum += pv[r];
                    v[i] = a.bias ? sum + bias_s[e] : sum;
                    a.ws.logits[(size_t)t * E + e] = v[i];
                } else {
                    v[i] = __ldg(a.logits_in + (size_t)t * E + e);
                }
            }
            RDEC_T(8)
            float sel_v[ROUTE_MAX_K];
            int sel_e[ROUTE_MAX_K];
            topk_warp<NVT>(v, taken, k, lane, sel_v, sel_e);
            RDEC_T(9)
            float my_v = sel_v[0];
            int my_e = 0;
#pragma unroll
            for (int j = 0; j < ROUTE_MAX_K; ++j)
                if (j == lane) { my_v = sel_v[j]; my_e = sel_e[j]; }
            const float my_ev = lane < k ? dx_expf(__fsub_rn(my_v, sel_v[0])) : 0.0f;
            float part_e[ROUTE_MAX_K];
#pragma unroll
            for (int j = 0; j < ROUTE_MAX_K; ++j) part_e[j] = __shfl_sync(0xffffffffu, my_ev, j);
            float sum = part_e[0];
#pragma unroll
            for (int j = 1; j < ROUTE_MAX_K; ++j)
                if (j < k) sum = __fadd_rn(sum, part_e[j]);
            if (lane < k) {
                const float gte = __fdiv_rn(my_ev, sum);
                const uint32_t gm = (uint32_t)rintf(__fmul_rn(gte, 16777216.0f));
                a.ws.idx[(size_t)t * k + lane] = my_e;
                a.ws.gate[(size_t)t * k + lane] = gte;
                a.ws.ent[t * k + lane] = (int16_t)my_e;
                const int le = my_e - a.e_lo;                   // a3: integer atomics, order-free (R-H1)
                if (a.cnt_acc && le >= 0 && le < a.e_cnt) {
                    atomicAdd(&a.cnt_acc[le], 1u);
                    atomicAdd(&a.mass_acc[le], (u64)gm);
                }
            }
        }
    }
    RDEC_T(10)
    if (a.wr && CS > 1) cluster_barrier();               // the cluster's partials are no longer read
    RDEC_T(3)
    for (int i = threadIdx.x; i < RDEC_CHUNKS * E; i += blockDim.x) chist[i] = 0;
    if ((int)gridDim.x == CS && CS > 1) cluster_barrier();  // T <= 16: the grid is one cluster
    else grid_sync(a.ws.gbar);
    RDEC_T(4)
    DX_GRID_LAUNCH();                       // every CTA is resident and past the barrier
    // ---------------- C: histograms, offsets, active list (every CTA, identical results)
    const int n = T * k;
    for (int i = threadIdx.x; i < n; i += blockDim.x) ent_s[i] = __ldcg(a.ws.ent + i);
    __syncthreads();
    {
        const int ci = warp, i = warp * 32 + lane;            // n <= 512 = 16 warps x 32 entries
        const bool have = i < n;
        const int ei = have ? ent_s[i] : -1 - lane;
        const unsigned same = __match_any_sync(0xffffffffu, ei);
        const int rk = __popc(same & ((1u << lane) - 1u));
        if (have) rk_s[i] = (int16_t)rk;
        if (have && rk == 0) chist[ci * E + ei] = (int16_t)__popc(same);
    }
    __syncthreads();
    const int e = threadIdx.x;                                // E <= 512 = blockDim
    uint32_t c = 0;
    if (e < E) {
#pragma unroll
        for (int c2 = 0; c2 < RDEC_CHUNKS; ++c2) c += (uint32_t)chist[c2 * E + e];
    }
    // one block scan of three packed 10-bit counts (every sum <= 512): rows, active experts, active HIGH experts;
    // the active list puts the HIGH tier first (the grouped GEMMs hand out work items in this order, heaviest first)
    const int32_t hi = (c && tier_e) ? 1 : 0;
    int32_t ptot;
    const int32_t pk = block_excl_scan<int32_t>((int32_t)c | ((c > 0 ? 1 : 0) << 10) | (hi << 20), tmp, &ptot);
    const int32_t o = pk & 1023, ac = (pk >> 10) & 1023, ah = (pk >> 20) & 1023;
    if (threadIdx.x == 0) { total_s = ptot & 1023; na_s = (ptot >> 10) & 1023; nhi_s = (ptot >> 20) & 1023; }
    __syncthreads();
    if (e < E) {
        if (blockIdx.x == 0) {
            a.ws.off[e] = o;
            if (c) a.ws.act_e[hi ? ah : nhi_s + (ac - ah)] = e;
        }
        int run = o;
#pragma unroll
        for (int c2 = 0; c2 < RDEC_CHUNKS; ++c2) {
            const int b = chist[c2 * E + e];
            chist[c2 * E + e] = (int16_t)run;
            run += b;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ws.off[E] = total_s;
        *a.ws.n_act = na_s;
        if (a.rs.stats && a.rs.tier) {                      // algorithmic weight bytes (profiling)
            const u64 nh = (u64)nhi_s, nl = (u64)na_s - nh;
            atomicAdd(&a.rs.stats[0], nh * a.rs.b10 + nl * a.rs.b00);
            atomicAdd(&a.rs.stats[1], nh * a.rs.b11 + nl * a.rs.b01);
            atomicAdd(&a.rs.stats[2], (u64)na_s);
        }
    }
    __syncthreads();
    RDEC_T(5)
    // a4: stable placement (pos = off[e] + earlier chunks + in-chunk rank) and the x-row gather, one warp
    // per entry, entries spread over all CTAs
    for (int i = warp * gridDim.x + blockIdx.x; i < n; i += gridDim.x * 16) {
        const int ei = ent_s[i];
        const int pos = chist[(i >> 5) * E + ei] + rk_s[i];
        if (lane == 0) {
            a.ws.perm[pos] = i;
            a.ws.inv[i] = pos;
        }
        if (a.Xp) {
            const uint4* src = reinterpret_cast<const uint4*>(a.x + (size_t)(i / k) * H);
            uint4* dst = reinterpret_cast<uint4*>(a.Xp + (size_t)pos * H);
            for (int h = lane; h < H / 8; h += 32) dst[h] = __ldg(src + h);
        }
    }
    RDEC_T(7)
#ifdef DX_RDEC_PROF
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0 && (atomicAdd(&g_rdec_n, 1) % 64) == 63)
        printf("rdec us: wait %.2f A %.2f B %.2f [logits %.2f topk %.2f rest %.2f cbar %.2f] sync %.2f C %.2f place %.2f total %.2f\n", (tstamp[1] - tstamp[0]) * 1e-3,
               (tstamp[2] - tstamp[1]) * 1e-3, (tstamp[3] - tstamp[2]) * 1e-3, (tstamp[8] - tstamp[2]) * 1e-3,
               (tstamp[9] - tstamp[8]) * 1e-3, (tstamp[10] - tstamp[9]) * 1e-3, (tstamp[3] - tstamp[10]) * 1e-3,
               (tstamp[4] - tstamp[3]) * 1e-3,
               (tstamp[5] - tstamp[4]) * 1e-3, (tstamp[7] - tstamp[5]) * 1e-3, (tstamp[7] - tstamp[0]) * 1e-3);
#endif
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

// a4 offsets, parallel over experts: block e scans expert e's per-route-block counts hist[e][0..nblk) into
// base[e][b] (rows of expert e in earlier route blocks) and its total; the last block to finish (completion
// counter) turns the totals into off[] (exclusive scan), the active-expert list (HIGH tier first: the grouped
// GEMMs hand out work items in this order, heaviest first) and the profiling byte counters.
__global__ void __launch_bounds__(256) k_scan_e(const int32_t* __restrict__ hist, int nblk, int E,
                                                int32_t* __restrict__ base, int32_t* __restrict__ off,
                                                int32_t* __restrict__ act_e, int32_t* __restrict__ n_act, RouteStats rs,
                                                unsigned* __restrict__ done) {
    __shared__ int32_t tmp[32];
    __shared__ int32_t total_s, na_s, nhi_s;
    __shared__ bool last;
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int e = blockIdx.x;
    int32_t run = 0;
    for (int b0 = 0; b0 < nblk; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        const int32_t v = b < nblk ? __ldcg(hist + (size_t)e * nblk + b) : 0;
        const int32_t x = block_excl_scan<int32_t>(v, tmp, &total_s);
        if (b < nblk) base[(size_t)e * nblk + b] = run + x;
        run += total_s;
    }
    if (threadIdx.x == 0) off[e] = run;                     // this expert's total, scanned below
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // E <= 512: two experts per thread
    const int e0 = 2 * threadIdx.x, e1 = e0 + 1;
    const int32_t t0 = e0 < E ? __ldcg(off + e0) : 0, t1 = e1 < E ? __ldcg(off + e1) : 0;
    const int32_t o = block_excl_scan<int32_t>(t0 + t1, tmp, &total_s);
    const int32_t a = block_excl_scan<int32_t>((t0 > 0) + (t1 > 0), tmp, &na_s);
    const bool h0 = e0 < E && t0 > 0 && rs.tier && rs.tier[e0], h1 = e1 < E && t1 > 0 && rs.tier && rs.tier[e1];
    const int32_t ah = block_excl_scan<int32_t>((int32_t)h0 + (int32_t)h1, tmp, &nhi_s);
    int32_t ahi = ah, alo = nhi_s + (a - ah);
    if (e0 < E) {
        off[e0] = o;
        if (t0 > 0) act_e[h0 ? ahi++ : alo++] = e0;
    }
    if (e1 < E) {
        off[e1] = o + t0;
        if (t1 > 0) act_e[h1 ? ahi++ : alo++] = e1;
    }
    if (rs.stats && rs.tier && threadIdx.x == 0) {          // algorithmic weight bytes of this forward (profiling)
        const u64 nh = (u64)nhi_s, nl = (u64)na_s - nh;
        atomicAdd(&rs.stats[0], nh * rs.b10 + nl * rs.b00);
        atomicAdd(&rs.stats[1], nh * rs.b11 + nl * rs.b01);
        atomicAdd(&rs.stats[2], (u64)na_s);
    }
    if (threadIdx.x == 0) { off[E] = total_s; *n_act = na_s; *done = 0; }
}

// One warp per entry (t*k + j): its row position = off[e] + rows of expert e in earlier route blocks
// (base[e][block]) + earlier entries of the same expert inside its route block -- the stable counting-sort
// order (t asc, j asc); the warp then copies x[t] into Xp[pos] (the B operand of the gate/up GEMM) when Xp != NULL.
__global__ void __launch_bounds__(256) k_place(const int32_t* __restrict__ idx, int n, int nblk, int k,
                                               const int32_t* __restrict__ base, const int32_t* __restrict__ off,
                                               int32_t* __restrict__ perm, int32_t* __restrict__ inv,
                                               const __nv_bfloat16* __restrict__ x, int H, __nv_bfloat16* __restrict__ Xp,
                                               const int32_t* __restrict__ rowmap) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= n) return;
    const int b = (i / k) / ROUTE_TOK_PER_BLK;
    const int e = __ldcg(idx + i);
    int r = 0;
    for (int q = b * ROUTE_TOK_PER_BLK * k + lane; q < i; q += 32) r += (__ldcg(idx + q) == e);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    const int pos = __ldcg(off + e) + __ldcg(base + (size_t)e * nblk + b) + r;
    if (lane == 0) {
        perm[pos] = i;
        inv[i] = pos;
    }
    if (!Xp) return;
    const int srow = rowmap ? __ldcg(rowmap + i) : i / k;        // f-2: deduplicated EP rows
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)srow * H);
    uint4* dst = reinterpret_cast<uint4*>(Xp + (size_t)pos * H);
    for (int h = lane; h < H / 8; h += 32) dst[h] = __ldg(src + h);
}

// ------------------------------------------------------------------ f-2 deduplicated EP dispatch
// Source side, after the routing over global experts and the placement (perm: entries sorted by expert, so owner d's
// entries are positions [off[d*E_loc], off[(d+1)*E_loc])): token t is sent to owner d ONCE however many of its k
// experts d owns.  mark[d][t] -> per-owner exclusive scan urow[d][t] (U_d rows) -> unique rows copied to the send
// buffer (owner blocks in order) -> per-entry metadata {local expert, gate bits, row within the owner block}.
__global__ void k_dedup_mark(const int32_t* __restrict__ idx, int n, int k, int E_loc, int T, int32_t* __restrict__ mark) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) mark[(size_t)(idx[i] / E_loc) * T + i / k] = 1;
}
__global__ void __launch_bounds__(256) k_dedup_scan(int32_t* __restrict__ mark, int T, const int32_t* __restrict__ off,
                                                    int E_loc, int32_t* __restrict__ triples, int T_src) {
    __shared__ int32_t tmp[32];
    __shared__ int32_t total_s;
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int d = blockIdx.x;
    int32_t run = 0;
    for (int t0 = 0; t0 < T; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        const int32_t v = t < T ? mark[(size_t)d * T + t] : 0;
        const int32_t x = block_excl_scan<int32_t>(v, tmp, &total_s);
        if (t < T) mark[(size_t)d * T + t] = v ? run + x : -1;      // row within owner d's block, -1: not sent
        run += total_s;
    }
    if (threadIdx.x == 0) {                                         // {unique rows, entries, my T} for owner d
        triples[3 * d] = run;
        triples[3 * d + 1] = off[(d + 1) * E_loc] - off[d * E_loc];
        triples[3 * d + 2] = T_src;
    }
}
__global__ void k_dedup_rows(const int32_t* __restrict__ urow, int T, int G, const int32_t* __restrict__ triples,
                             const __nv_bfloat16* __restrict__ x, int H, __nv_bfloat16* __restrict__ send_rows) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int lane = threadIdx.x & 31;
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= G * T) return;
    const int d = w / T, t = w % T;
    const int r = urow[(size_t)d * T + t];
    if (r < 0) return;
    int base = 0;
    for (int q = 0; q < d; ++q) base += triples[3 * q];
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * H);
    uint4* dst = reinterpret_cast<uint4*>(send_rows + (size_t)(base + r) * H);
    for (int h = lane; h < H / 8; h += 32) dst[h] = __ldg(src + h);
}
__global__ void k_dedup_meta(const int32_t* __restrict__ perm, const int32_t* __restrict__ idx,
                             const float* __restrict__ gate, const int32_t* __restrict__ urow, int n, int k, int E_loc,
                             int T, int4* __restrict__ meta) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= n) return;
    const int i = perm[pos];
    const int e = idx[i];
    const int d = e / E_loc;
    meta[pos] = make_int4(e % E_loc, __float_as_int(gate[i]), urow[(size_t)d * T + i / k], 0);
}
// Owner side: received entries meta4[R] (in source order) with rows relative to their source's block; sources' entry
// and row offsets in `so` ({entry offset, row offset} per source, G + 1 entries) -> meta2 {expert, gate} for the
// owner-side routing and rowmap[i] = the entry's row among the received rows.
struct SrcOffs {
    int32_t e[9], r[9];
};
__global__ void k_dedup_fix(const int4* __restrict__ meta4, int R, int G, SrcOffs so, int2* __restrict__ meta2,
                            int32_t* __restrict__ rowmap) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= R) return;
    int s = 0;
    while (s + 1 < G && i >= so.e[s + 1]) ++s;
    const int4 m = meta4[i];
    meta2[i] = make_int2(m.x, m.y);
    rowmap[i] = so.r[s] + m.z;
}


// ------------------------------------------------------------------ f-3 shared expert rows (Eq. 1 first sum)
// After routing: entries n .. n+T-1 (n = T*k) are the shared expert's rows, one per token in order: perm, gate 1.0
// (bf16(1 * o) = bf16(o) exactly), Xp[n + t] = x[t]; off[E + 1] = n + T; the shared expert (id E) goes first in the
// active list (the heaviest item); its algorithmic weight bytes join the profiling counters.  Block 0 rewrites the
// active list; every block copies a share of the rows.
__global__ void __launch_bounds__(256) k_shared_rows(int32_t* __restrict__ perm, float* __restrict__ gate,
                                                     int32_t* __restrict__ off, int32_t* __restrict__ act_e,
                                                     int32_t* __restrict__ n_act, u64* __restrict__ stats, u64 b0, u64 b1,
                                                     int T, int k, int E, int H, const __nv_bfloat16* __restrict__ x,
                                                     __nv_bfloat16* __restrict__ Xp) {
    __shared__ int32_t lst[ROUTE_MAX_E];
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int n = T * k;
    if (blockIdx.x == 0) {
        const int na = *n_act;
        for (int i = threadIdx.x; i < na; i += blockDim.x) lst[i] = act_e[i];
        __syncthreads();
        for (int i = threadIdx.x; i < na; i += blockDim.x) act_e[i + 1] = lst[i];
        if (threadIdx.x == 0) {
            act_e[0] = E;
            *n_act = na + 1;
            off[E + 1] = n + T;
            if (stats) {
                atomicAdd(&stats[0], b0);
                atomicAdd(&stats[1], b1);
                atomicAdd(&stats[2], 1ull);
            }
        }
    }
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
        perm[n + t] = n + t;
        gate[n + t] = 1.0f;
    }
    if (!Xp) return;
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    for (int t = blockIdx.x * wpb + (threadIdx.x >> 5); t < T; t += gridDim.x * wpb) {
        const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * H);
        uint4* dst = reinterpret_cast<uint4*>(Xp + (size_t)(n + t) * H);
        for (int h = lane; h < H / 8; h += 32) dst[h] = __ldg(src + h);
    }
}

// ------------------------------------------------------------------ a8: y_t = bf16(sum_j Y[t,j])
// inv == NULL: Y rows in entry order (t*k + j); else Y rows in permuted order, entry i at row inv[i]
// (expert-parallel combine: the rows come back from their owners in dispatch order).  Block = (token,
// segment of 8*blockDim columns); every row load of a thread is issued before the rank-order fp32 sum.
// fold_on: the LAST block instead runs the layer's EMA fold + publication (a10, a14), after the down GEMM
// finished (griddepcontrol.wait), so the table flip never races the GEMMs that read the tables.
__global__ void __launch_bounds__(128) k_combine(const __nv_bfloat16* __restrict__ Y, int k, int H, int nseg, int cthr,
                                                 __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ inv,
                                                 const Ctrl c, int fold_on, int fold_layer_id, u64 B_tot, double oma,
                                                 int shared_base) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    if (fold_on && blockIdx.x == gridDim.x - 1) {
        fold_layer(c, fold_layer_id, B_tot, oma);
        return;
    }
    if ((int)threadIdx.x >= cthr) return;
    const int t = blockIdx.x / nseg, seg = blockIdx.x % nseg;
    const int h = (seg * cthr + threadIdx.x) * 8;
    uint4 v[ROUTE_MAX_K];
#pragma unroll
    for (int j = 0; j < ROUTE_MAX_K; ++j) {
        if (j < k) {
            const size_t row = inv ? (size_t)inv[(size_t)t * k + j] : (size_t)t * k + j;
            v[j] = __ldcg(reinterpret_cast<const uint4*>(Y + row * H + h));
        }
    }
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
    if (shared_base >= 0) {                      // f-3: the shared expert's term first (R-S1)
        const uint4 vs = __ldcg(reinterpret_cast<const uint4*>(Y + ((size_t)shared_base + t) * H + h));
        const uint16_t* b = reinterpret_cast<const uint16_t*>(&vs);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], dx_bf2f(b[i]));
    }
#pragma unroll
    for (int j = 0; j < ROUTE_MAX_K; ++j) {
        if (j < k) {
            const uint16_t* b = reinterpret_cast<const uint16_t*>(&v[j]);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], dx_bf2f(b[i]));
        }
    }
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16_rn(acc[i]);
    *reinterpret_cast<uint4*>(y + (size_t)t * H + h) = *reinterpret_cast<const uint4*>(o);
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
            idx_out[r] = 0;                                  // a valid placement with a zero gate
            gate_out[r] = 0.0f;
            atomicAdd(&cnt_s[0], 1u);
        } else {
            idx_out[r] = m.x;
            gate_out[r] = g;
            atomicAdd(&cnt_s[m.x], 1u);
            atomicAdd(&mass_s[m.x], (u64)rintf(__fmul_rn(g, 16777216.0f)));
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        hist[(size_t)e * gridDim.x + blockIdx.x] = (int32_t)cnt_s[e];     // [expert][route block]
        if (cnt_s[e] && cnt_acc) {
            atomicAdd(&cnt_acc[e], cnt_s[e]);
            atomicAdd(&mass_acc[e], mass_s[e]);
        }
    }
}

// Source side after placement: metadata of every dispatched row (local expert id at its owner, gate
// bits) and per-owner row counts (rows for owner o are contiguous because experts are partitioned
// contiguously: [off[o*E_loc], off[(o+1)*E_loc]) ).
__global__ void k_ep_meta(const int32_t* __restrict__ perm, const int32_t* __restrict__ idx,
                          const float* __restrict__ gate, const int32_t* __restrict__ off, int n, int E_loc, int G,
                          int2* __restrict__ meta, int32_t* __restrict__ counts, int2* __restrict__ pairs, int T_src) {
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos < n) {
        const int ent = perm[pos];
        const int e = idx[ent];
        meta[pos] = make_int2(e % E_loc, __float_as_int(gate[ent]));
    }
    if (pos < G) {
        const int c = off[(pos + 1) * E_loc] - off[pos * E_loc];
        if (counts) counts[pos] = c;
        if (pairs) pairs[pos] = make_int2(c, T_src);     // {rows for owner pos, my token count} (NCCL transport)
    }
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
    if (T >= 128 && H % RT_K == 0) {               // prefill-sized batches: the tiled GEMM
        dim3 grid((T + RT_M - 1) / RT_M, (E + RT_N - 1) / RT_N);
        dx_launch(k_router_tiled, grid, dim3(256), 0, st, g_dx_pdl, x, wr, bias, T, E, H, logits);
        return;
    }
    dim3 grid((E + 7) / 8, (T + 15) / 16);
    dx_launch(k_router, grid, dim3(512), 0, st, g_dx_pdl, x, wr, bias, T, E, H, logits);
}

static void launch_scan_e(int nblk, int E, const RouteWs& ws, const RouteStats& rs, cudaStream_t st);

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
    launch_scan_e(nb, E, ws, rs, st);
}

bool route_dec_ok(int T, int E, int k) {
    // T <= 128: at most 8 clusters of 8 CTAs, so the grid barrier's CTAs are always co-resident
    return T >= 1 && T <= 128 && T * k <= RDEC_MAX_ENT && E <= 512 && E % 32 == 0 && k <= ROUTE_MAX_K;
}

template <int NVT>
static void launch_rdec(const RouteDecArgs& a, int grid, size_t smem, cudaStream_t st) {
    static unsigned long long attr_mask = 0;
    if (dx_first_on_device(attr_mask))
        cudaFuncSetAttribute(k_route_dec<NVT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = a.cs;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
    if (g_dx_pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, k_route_dec<NVT>, a);
}

void launch_route_dec(const __nv_bfloat16* x, const __nv_bfloat16* wr, const float* bias, const float* logits_in,
                      int T, int E, int k, int H, int e_lo, const RouteWs& ws, uint32_t* cnt_acc, u64* mass_acc,
                      const int32_t* tier, const u64 (&bytes)[2][2], __nv_bfloat16* Xp, cudaStream_t st) {
    if (T <= 0) return;
    RouteDecArgs a;
    a.x = x; a.wr = wr; a.bias = bias; a.logits_in = logits_in;
    a.T = T; a.E = E; a.k = k; a.H = H; a.e_lo = e_lo; a.e_cnt = cnt_acc ? E : 0;
    a.ws = ws; a.cnt_acc = cnt_acc; a.mass_acc = mass_acc;
    a.rs = RouteStats{tier, bytes[0][0], bytes[0][1], bytes[1][0], bytes[1][1], ws.stats};
    a.Xp = Xp;
    // clusters of cs CTAs per 16-token tile (router mode: they split K, each slice a multiple of 16)
    int cs = 8;
    if (wr)
        while (cs > 1 && H % (16 * cs) != 0) cs >>= 1;
    a.cs = cs;
    const int pitch = H / cs + 8;                       // staged row (bf16) of the router slices
    int ech = E;                                        // experts staged per round (W_r slice rows)
    while (ech > 128 && (size_t)(16 + ech) * pitch * 2 > 96 * 1024) ech >>= 1;
    a.ech = ech;
    const int grid = ((T + 15) / 16) * cs;
    size_t smem = (size_t)E * 16 * 4 > (size_t)RDEC_CHUNKS * E * 2 ? (size_t)E * 16 * 4 : (size_t)RDEC_CHUNKS * E * 2;
    if (wr) smem = (size_t)E * 16 * 4 + (size_t)(16 + ech) * pitch * 2;
    if (E <= 128)      launch_rdec<4>(a, grid, smem, st);
    else if (E <= 256) launch_rdec<8>(a, grid, smem, st);
    else               launch_rdec<16>(a, grid, smem, st);
}

void launch_place(int T, int E, int k, const RouteWs& ws, const __nv_bfloat16* x, int H, __nv_bfloat16* Xp,
                  cudaStream_t st, const int32_t* rowmap) {
    if (T <= 0) return;
    const int n = T * k;
    dx_launch(k_place, dim3((n + 7) / 8), dim3(256), 0, st, g_dx_pdl, (const int32_t*)ws.idx, n, route_blocks(T), k,
              (const int32_t*)ws.base, (const int32_t*)ws.off, ws.perm, ws.inv, x, H, Xp, rowmap);
}

void launch_dedup_dispatch(const RouteWs& ws, int T, int k, int E_loc, int G, const __nv_bfloat16* x, int H,
                           int32_t* mark, int32_t* triples, __nv_bfloat16* send_rows, int4* meta, cudaStream_t st) {
    if (T <= 0) return;
    const int n = T * k;
    cudaMemsetAsync(mark, 0, (size_t)G * T * sizeof(int32_t), st);
    dx_launch(k_dedup_mark, dim3((n + 255) / 256), dim3(256), 0, st, g_dx_pdl, (const int32_t*)ws.idx, n, k, E_loc, T, mark);
    dx_launch(k_dedup_scan, dim3(G), dim3(256), 0, st, g_dx_pdl, mark, T, (const int32_t*)ws.off, E_loc, triples, T);
    dx_launch(k_dedup_rows, dim3((G * T + 7) / 8), dim3(256), 0, st, g_dx_pdl, (const int32_t*)mark, T, G,
              (const int32_t*)triples, x, H, send_rows);
    dx_launch(k_dedup_meta, dim3((n + 255) / 256), dim3(256), 0, st, g_dx_pdl, (const int32_t*)ws.perm,
              (const int32_t*)ws.idx, (const float*)ws.gate, (const int32_t*)mark, n, k, E_loc, T, meta);
}

void launch_dedup_fix(const int4* meta4, int R, int G, const int32_t* eoff, const int32_t* roff, int2* meta2,
                      int32_t* rowmap, cudaStream_t st) {
    if (R <= 0) return;
    SrcOffs so{};
    for (int s = 0; s <= G && s < 9; ++s) { so.e[s] = eoff[s]; so.r[s] = roff[s]; }
    dx_launch(k_dedup_fix, dim3((R + 255) / 256), dim3(256), 0, st, g_dx_pdl, meta4, R, G, so, meta2, rowmap);
}

void launch_shared_rows(const RouteWs& ws, int T, int k, int E, int H, const __nv_bfloat16* x, __nv_bfloat16* Xp,
                        u64 b0, u64 b1, cudaStream_t st) {
    if (T <= 0) return;
    const int blocks = (T + 7) / 8 < 148 ? (T + 7) / 8 : 148;
    dx_launch(k_shared_rows, dim3(blocks), dim3(256), 0, st, g_dx_pdl, ws.perm, ws.gate, ws.off, ws.act_e, ws.n_act,
              ws.stats, b0, b1, T, k, E, H, x, Xp);
}

static void launch_scan_e(int nblk, int E, const RouteWs& ws, const RouteStats& rs, cudaStream_t st) {
    dx_launch(k_scan_e, dim3(E), dim3(256), 0, st, g_dx_pdl, (const int32_t*)ws.hist, nblk, E, ws.base, ws.off,
              ws.act_e, ws.n_act, rs, ws.done);
}

void launch_combine(const __nv_bfloat16* Y, int T, int k, int H, __nv_bfloat16* y, cudaStream_t st,
                    const int32_t* inv, const Ctrl* ctrl, const FoldReq* fold, int shared_base) {
    if (T <= 0 && !fold) return;
    int nseg = 1;                               // segments of <= 128 threads x 8 columns that tile H exactly
    while ((H / 8) / nseg > 128 || (H / 8) % nseg) ++nseg;
    const int cthr = (H / 8) / nseg;
    const int blocks = T * nseg + (fold ? 1 : 0);
    Ctrl c{};
    if (ctrl) c = *ctrl;
    const int threads = fold ? (cthr > 128 ? cthr : 128) : cthr;
    dx_launch(k_combine, dim3(blocks), dim3(threads), 0, st, g_dx_pdl, Y, k, H, nseg, cthr, y,
              inv, c, fold ? 1 : 0, fold ? fold->layer : 0, fold ? fold->B_tot : (u64)0,
              ctrl ? 1.0 - ctrl->alpha : 0.0, shared_base);
}

void launch_route_given(const int2* meta, int R, int E, const RouteWs& ws, uint32_t* cnt_acc, u64* mass_acc,
                        const int32_t* tier, const u64 (&bytes)[2][2], int32_t* err, cudaStream_t st) {
    if (R <= 0) return;
    RouteStats rs{tier, bytes[0][0], bytes[0][1], bytes[1][0], bytes[1][1], ws.stats};
    dx_launch(k_route_given, dim3(route_blocks(R)), dim3(256), 0, st, g_dx_pdl, meta, R, E, ws.idx, ws.gate, ws.hist,
              cnt_acc, mass_acc, ws.base, ws.off, ws.act_e, ws.n_act, rs, ws.done, err);
    launch_scan_e(route_blocks(R), E, ws, rs, st);
}

void launch_ep_meta(const RouteWs& ws, int n, int E_loc, int G, int2* meta, int32_t* counts, int2* pairs, int T_src,
                    cudaStream_t st) {
    const int thr = 256, nb = ((n > G ? n : G) + thr - 1) / thr;
    dx_launch(k_ep_meta, dim3(nb > 0 ? nb : 1), dim3(thr), 0, st, g_dx_pdl, (const int32_t*)ws.perm,
              (const int32_t*)ws.idx, (const float*)ws.gate, (const int32_t*)ws.off, n, E_loc, G, meta, counts, pairs, T_src);
}

void launch_counts_from(const int32_t* idx, const float* gate, int T, int E, int e_cnt, int k, int e_lo,
                        uint32_t* cnt_acc, u64* mass_acc, int32_t* err, cudaStream_t st) {
    if (T <= 0) return;
    k_counts_from<<<(T + 127) / 128, 128, 0, st>>>(idx, gate, T, E, k, e_lo, e_cnt, cnt_acc, mass_acc, err);
}
