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
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
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
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (e >= E) return;
    const __nv_bfloat16* row = wr + (size_t)e * H;
    float acc[TT];
#pragma unroll
    for (int t = 0; t < TT; ++t) acc[t] = 0.0f;
#pragma unroll 8
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
    int32_t ai = a;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int e = h ? e1 : e0;
        const int32_t tot = h ? t1 : t0;
        if (e >= E) continue;
        const int32_t oe = h ? o + t0 : o;
        off[e] = oe;
        if (tot > 0) {
            act_e[ai++] = e;
            if (rs.stats && rs.tier) {          // algorithmic weight bytes of this forward (profiling)
                const int ti = rs.tier[e];
                atomicAdd(&rs.stats[0], ti ? rs.b10 : rs.b00);
                atomicAdd(&rs.stats[1], ti ? rs.b11 : rs.b01);
                atomicAdd(&rs.stats[2], 1ull);
            }
        }
        int32_t run = oe;
        for (int b = 0; b < nblk; ++b) {
            base[(size_t)b * E + e] = run;
            run += __ldcg(hist + (size_t)b * E + e);
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

void launch_router(const __nv_bfloat16* x, const __nv_bfloat16* wr, const float* bias, int T, int E,
                   int H, float* logits, cudaStream_t st) {
    if (T <= 0) return;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_router<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_router<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    // 4 warps (experts) per block: decode batches still spread the 4 KB router rows over >= 32 blocks
    if (T <= 4) {
        dim3 grid((E + 3) / 4, (T + 3) / 4);
        dx_launch(k_router<4>, grid, dim3(128), 4 * H * sizeof(float), st, g_dx_pdl, x, wr, bias, T, E, H, logits);
    } else {
        dim3 grid((E + 3) / 4, (T + 7) / 8);
        dx_launch(k_router<8>, grid, dim3(128), 8 * H * sizeof(float), st, g_dx_pdl, x, wr, bias, T, E, H, logits);
    }
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
