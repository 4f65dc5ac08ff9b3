// k_route.cu -- router logits (a1), warp-shuffle top-k + softmax gates + hotness counters (a2, a3),
// stable permutation by expert (a4) and the weighted combine (a8).
//   Eq. 1: K = topk({g_i(x)}), y = sum_{j in K} g_j E_j(x).
//   "records the selected experts and accumulates gating probabilities".
// Readings: R-G1 (ties -> lower id, gates = softmax over the k selected logits), R-G2 (dx_expf),
// R-H1 (cnt u32, mass = sum rint(g * 2^24) u64: integer sums are order-free => bit-exact).
#include "dx_common.cuh"

#define ROUTE_TOK_PER_BLK 8
#define ROUTE_MAX_E 512
#define ROUTE_MAX_K 16

namespace {

// ------------------------------------------------------------------ a1: logits = x Wr^T (+b), fp32
template <int TT>
__global__ void __launch_bounds__(256) k_router(const __nv_bfloat16* __restrict__ x,
                                                const __nv_bfloat16* __restrict__ wr,
                                                const float* __restrict__ bias, int T, int E, int H,
                                                float* __restrict__ logits) {
    extern __shared__ float xs[];   // [TT][H]
    const int t0 = blockIdx.y * TT;
    const int nt = min(TT, T - t0);
    for (int i = threadIdx.x; i < TT * H / 8; i += blockDim.x) {
        const int t = (i * 8) / H, h = (i * 8) % H;
        float* d = xs + t * H + h;
        if (t < nt) {
            uint4 v = *reinterpret_cast<const uint4*>(x + (size_t)(t0 + t) * H + h);
            const uint16_t* b = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
            for (int j = 0; j < 8; ++j) d[j] = dx_bf2f(b[j]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) d[j] = 0.0f;
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int e = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (e >= E) return;
    const __nv_bfloat16* row = wr + (size_t)e * H;
    float acc[TT];
#pragma unroll
    for (int t = 0; t < TT; ++t) acc[t] = 0.0f;
    for (int k = lane * 8; k < H; k += 256) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>(row + k));
        const uint16_t* b = reinterpret_cast<const uint16_t*>(&v);
        float w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = dx_bf2f(b[j]);
#pragma unroll
        for (int t = 0; t < TT; ++t) {
            const float4 a = *reinterpret_cast<const float4*>(xs + t * H + k);
            const float4 c = *reinterpret_cast<const float4*>(xs + t * H + k + 4);
            acc[t] = fmaf(w[0], a.x, acc[t]); acc[t] = fmaf(w[1], a.y, acc[t]);
            acc[t] = fmaf(w[2], a.z, acc[t]); acc[t] = fmaf(w[3], a.w, acc[t]);
            acc[t] = fmaf(w[4], c.x, acc[t]); acc[t] = fmaf(w[5], c.y, acc[t]);
            acc[t] = fmaf(w[6], c.z, acc[t]); acc[t] = fmaf(w[7], c.w, acc[t]);
        }
    }
#pragma unroll
    for (int t = 0; t < TT; ++t) {
        float v = acc[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && t < nt) logits[(size_t)(t0 + t) * E + e] = v + (bias ? bias[e] : 0.0f);
    }
}

__device__ __forceinline__ bool better(float a, int ea, float b, int eb) {
    return a > b || (a == b && ea < eb);
}

// ------------------------------------------------------------------ a2 + a3: top-k, gates, counters
// One warp per token (8 tokens per block), k rounds of (value desc, id asc) warp arg-max over NVT
// logits per lane; per-block shared histograms merged into the layer's global accumulators with one
// atomic per touched expert.
template <int NVT>
__global__ void __launch_bounds__(256) k_route(const float* __restrict__ logits, int T, int E, int k,
                                               int e_lo, int e_cnt, int32_t* __restrict__ idx_out,
                                               float* __restrict__ gate_out, int32_t* __restrict__ hist,
                                               uint32_t* __restrict__ cnt_acc, u64* __restrict__ mass_acc) {
    __shared__ uint32_t cnt_s[ROUTE_MAX_E];
    __shared__ u64 mass_s[ROUTE_MAX_E];
    for (int e = threadIdx.x; e < E; e += blockDim.x) { cnt_s[e] = 0; mass_s[e] = 0; }
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
#pragma unroll
        for (int j = 0; j < ROUTE_MAX_K; ++j) {
            if (j >= k) break;
            float bv = -INFINITY;
            int be = 0x7fffffff;
#pragma unroll
            for (int i = 0; i < NVT; ++i) {
                const int e = lane + 32 * i;
                if (!((taken >> i) & 1u) && better(v[i], e, bv, be)) { bv = v[i]; be = e; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oe = __shfl_xor_sync(0xffffffffu, be, o);
                if (better(ov, oe, bv, be)) { bv = ov; be = oe; }
            }
            if ((be & 31) == lane) taken |= 1u << (be >> 5);
            sel_v[j] = bv;
            sel_e[j] = be;
        }
        // gates: softmax over the selected logits, sequential fp32 sum in rank order (R-G2)
        float ev[ROUTE_MAX_K];
        float sum = 0.0f;
#pragma unroll
        for (int j = 0; j < ROUTE_MAX_K; ++j) {
            if (j >= k) break;
            ev[j] = dx_expf(__fsub_rn(sel_v[j], sel_v[0]));
            sum = (j == 0) ? ev[0] : __fadd_rn(sum, ev[j]);
        }
#pragma unroll
        for (int j = 0; j < ROUTE_MAX_K; ++j) {
            if (j >= k) break;
            if (lane == j) {
                const float gte = __fdiv_rn(ev[j], sum);
                idx_out[(size_t)t * k + j] = sel_e[j];
                gate_out[(size_t)t * k + j] = gte;
                atomicAdd(&cnt_s[sel_e[j]], 1u);
                atomicAdd(&mass_s[sel_e[j]], (u64)rintf(__fmul_rn(gte, 16777216.0f)));
            }
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

// single block of 512 threads: E <= 512
__global__ void __launch_bounds__(512) k_scan(const int32_t* __restrict__ hist, int nblk, int E,
                                              int32_t* __restrict__ base, int32_t* __restrict__ off,
                                              int32_t* __restrict__ act_e, int32_t* __restrict__ n_act,
                                              const int32_t* __restrict__ tier, u64 b00, u64 b01, u64 b10,
                                              u64 b11, u64* __restrict__ stats) {
    __shared__ int32_t tmp[32];
    __shared__ int32_t tot_s, na_s;
    const int e = threadIdx.x;
    int32_t tot = 0;
    if (e < E)
        for (int b = 0; b < nblk; ++b) tot += hist[(size_t)b * E + e];
    int32_t total;
    const int32_t o = block_excl_scan<int32_t>(e < E ? tot : 0, tmp, &total);
    const int32_t a = block_excl_scan<int32_t>((e < E && tot > 0) ? 1 : 0, tmp, &na_s);
    if (e < E) {
        off[e] = o;
        if (tot > 0) {
            act_e[a] = e;
            if (stats && tier) {          // algorithmic weight bytes of this forward (profiling)
                const int ti = tier[e];
                atomicAdd(&stats[0], ti ? b10 : b00);
                atomicAdd(&stats[1], ti ? b11 : b01);
                atomicAdd(&stats[2], 1ull);
            }
        }
        int32_t run = o;
        for (int b = 0; b < nblk; ++b) {
            base[(size_t)b * E + e] = run;
            run += hist[(size_t)b * E + e];
        }
    }
    if (threadIdx.x == 0) { off[E] = total; *n_act = na_s; }
    (void)tot_s;
}

// one thread per entry (t*k + j): position = base[block][e] + number of earlier entries of the same
// expert inside its route block (<= 8k comparisons): the stable counting-sort order (t asc, j asc).
__global__ void __launch_bounds__(256) k_scatter(const int32_t* __restrict__ idx, int T, int E, int k,
                                                 const int32_t* __restrict__ base,
                                                 int32_t* __restrict__ perm, int32_t* __restrict__ inv) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T * k) return;
    const int b = (i / k) / ROUTE_TOK_PER_BLK;
    const int e = idx[i];
    int r = 0;
    for (int q = b * ROUTE_TOK_PER_BLK * k; q < i; ++q) r += (idx[q] == e);
    const int pos = base[(size_t)b * E + e] + r;
    perm[pos] = i;
    inv[i] = pos;
}

// ------------------------------------------------------------------ a8: y_t = bf16(sum_j Y[t,j])
__global__ void k_combine(const __nv_bfloat16* __restrict__ Y, int k, int H, __nv_bfloat16* __restrict__ y) {
    const int t = blockIdx.x;
    for (int h = threadIdx.x * 8; h < H; h += blockDim.x * 8) {
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
        for (int j = 0; j < k; ++j) {
            uint4 v = *reinterpret_cast<const uint4*>(Y + ((size_t)t * k + j) * H + h);
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

void launch_router(const __nv_bfloat16* x, const __nv_bfloat16* wr, const float* bias, int T, int E,
                   int H, float* logits, cudaStream_t st) {
    if (T <= 0) return;
    if (T <= 4) {
        dim3 grid((E + 7) / 8, (T + 3) / 4);
        k_router<4><<<grid, 256, 4 * H * sizeof(float), st>>>(x, wr, bias, T, E, H, logits);
    } else {
        dim3 grid((E + 7) / 8, (T + 7) / 8);
        size_t sm = 8 * H * sizeof(float);
        static bool attr = false;
        if (!attr) { cudaFuncSetAttribute(k_router<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); attr = true; }
        k_router<8><<<grid, 256, sm, st>>>(x, wr, bias, T, E, H, logits);
    }
}

void launch_route(const float* logits, int T, int E, int k, int e_lo, const RouteWs& ws,
                  uint32_t* cnt_acc, u64* mass_acc, cudaStream_t st) {
    (void)e_lo;
    if (T <= 0) return;
    const int nb = route_blocks(T), ec = cnt_acc ? E : 0;
    if (E <= 128)      k_route<4><<<nb, 256, 0, st>>>(logits, T, E, k, e_lo, ec, ws.idx, ws.gate, ws.hist, cnt_acc, mass_acc);
    else if (E <= 256) k_route<8><<<nb, 256, 0, st>>>(logits, T, E, k, e_lo, ec, ws.idx, ws.gate, ws.hist, cnt_acc, mass_acc);
    else               k_route<16><<<nb, 256, 0, st>>>(logits, T, E, k, e_lo, ec, ws.idx, ws.gate, ws.hist, cnt_acc, mass_acc);
}

void launch_scan_scatter(int T, int E, int k, const RouteWs& ws, const int32_t* tier, const u64 (&bytes)[2][2],
                         cudaStream_t st) {
    if (T <= 0) return;
    const int nblk = route_blocks(T);
    k_scan<<<1, 512, 0, st>>>(ws.hist, nblk, E, ws.base, ws.off, ws.act_e, ws.n_act, tier, bytes[0][0],
                              bytes[0][1], bytes[1][0], bytes[1][1], ws.stats);
    k_scatter<<<(T * k + 255) / 256, 256, 0, st>>>(ws.idx, T, E, k, ws.base, ws.perm, ws.inv);
}

void launch_combine(const __nv_bfloat16* Y, int T, int k, int H, __nv_bfloat16* y, cudaStream_t st) {
    if (T <= 0) return;
    int threads = H / 8 < 256 ? H / 8 : 256;
    k_combine<<<T, threads, 0, st>>>(Y, k, H, y);
}

void launch_counts_from(const int32_t* idx, const float* gate, int T, int E, int k, int e_lo,
                        uint32_t* cnt_acc, u64* mass_acc, int32_t* err, cudaStream_t st) {
    if (T <= 0) return;
    k_counts_from<<<(T + 127) / 128, 128, 0, st>>>(idx, gate, T, E, k, e_lo, E, cnt_acc, mass_acc, err);
}
