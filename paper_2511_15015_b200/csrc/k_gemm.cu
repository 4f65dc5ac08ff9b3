// k_gemm.cu -- tcgen05 grouped expert GEMMs over the slot pool (a6 gate/up + SwiGLU, a7 down + gate
// scaling), one persistent kernel per phase, every touched expert at its stable tier.
//   Eq. 1: E_j(x) = W_down (silu(W_gate x) * W_up x).
//
// Swap-AB: the weights are the M = 128 operand, the tokens of one expert are N (16..128, chosen per
// chunk from the expert's token count), the accumulator D[128 x N] fp32 lives in TMEM (two buffers, so
// the epilogue of one chunk overlaps the MMAs of the next).  Persistent CTAs (one per SM) walk the work
// items (expert, 128-row block) round-robin.
//
// Stage ring (6 x 32 KB smem): an A region (16 KB) and a B region (16 KB).  A bf16 stage holds one
// 64-wide K chunk: A = 128 weight rows TMA'd straight into the 128 B-swizzled UMMA layout.  A quantised
// stage holds KS = 4 (int4) or 8 (int2) K chunks of raw codes (16 KB), so every stage carries 16 KB of
// weight bytes whatever the tier (the HBM stream stays deep), with KS B sub-tiles.  Raw codes are
// dequantised exactly (bf16_rn((q-z)s), R-Q1) by two transform warp groups straight into a ring of
// 32-column TMEM A buffers (lane = weight row) that feeds tcgen05.mma with A in tensor memory.
// Gate/up items take 64 gate rows (A rows 0-63) and the matching 64 up rows (64-127); the SwiGLU pairs
// meet through a small smem exchange in the epilogue.
// Warp roles (448 threads): 0 TMA producer, 1 TMEM owner + MMA issuer, 2-9 transform, 10-13 epilogue.
#include "dx_common.cuh"
#include "dx_sm100.cuh"

using namespace sm100;

namespace {

constexpr int GEMM_THREADS = 448;
constexpr int KCH = 64;                       // K elements per chunk (128 B of bf16 per row)
constexpr int STAGES = 6;
constexpr int A_BYTES = 128 * 128;            // A / raw region per stage
constexpr int B_REGION = 16384;               // B region per stage
constexpr int STAGE_BYTES = A_BYTES + B_REGION;
constexpr int XCH_BYTES = 64 * 32 * 4;        // epilogue SwiGLU exchange: 64 rows x 32 columns fp32

// DEC: decode configuration (T <= 64): N <= 64 for bf16, 32 for int4, 16 for int2 with KS chunks per
// quantised stage; otherwise (prefill) N <= 128 and one chunk per stage for every tier.
template <bool DEC>
struct Cfg {
    static constexpr int NBMAX = DEC ? 64 : 128;
    static constexpr int NA = (512 - 2 * NBMAX) / 32;          // TMEM A buffers (32 columns each)
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + XCH_BYTES + 2048 + 2 * 128 * 17 * 4;
    __device__ static int nb(int bits) { return DEC ? (bits == 16 ? 64 : (bits == 4 ? 32 : 16)) : 128; }
    __device__ static int ks(int bits) { return (DEC && bits != 16) ? 16 / bits : 1; }   // int4: 4, int2: 8
};

__device__ __forceinline__ uint32_t bf2_sub_mul(uint32_t v, uint32_t zz, uint32_t ss) {
    __nv_bfloat162 r = __hmul2(__hsub2(*reinterpret_cast<__nv_bfloat162*>(&v), *reinterpret_cast<__nv_bfloat162*>(&zz)),
                               *reinterpret_cast<__nv_bfloat162*>(&ss));
    return *reinterpret_cast<uint32_t*>(&r);
}

// Decoded work item: expert e, 128-row block mb, its token rows [r0, r0+m), tier / slot / bits.
struct Item {
    int e, mb, r0, m, ti, slot, bits;
};
__device__ __forceinline__ Item decode(const GemmArgs& a, int item, int nmb) {
    Item it;
    it.e = a.act_e[item / nmb];
    it.mb = item % nmb;
    it.r0 = a.off[it.e];
    it.m = a.off[it.e + 1] - it.r0;
    it.ti = a.tier[it.e];
    it.slot = a.slot[it.e];
    it.bits = it.ti ? a.hi.bits : a.lo.bits;
    return it;
}

__device__ __forceinline__ int box_rows(int nvalid) {        // B tile rows: power of two in [16, 128]
    int r = 16;
    while (r < nvalid) r <<= 1;
    return r;
}

template <int PHASE, bool DEC>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_gemm(const __grid_constant__ GemmMaps maps, GemmArgs a) {
    using C = Cfg<DEC>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sS = smem;                                   // [STAGES][A 16 KB | B 16 KB]
    float* xch = reinterpret_cast<float*>(sS + STAGES * STAGE_BYTES);            // [32 cols][64 rows]
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xch) + XCH_BYTES);
    uint64_t* full = bars;                                // [STAGES] TMA landed (A or raw, and B)
    uint64_t* empty = full + STAGES;                      // [STAGES] MMA finished with the stage
    uint64_t* aready = empty + STAGES;                    // [NA] transform wrote TMEM A buffer
    uint64_t* aempty = aready + C::NA;                    // [NA] MMA finished with TMEM A buffer
    uint64_t* tfull = aempty + C::NA;                     // [2] accumulator ready
    uint64_t* tempty = tfull + 2;                         // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int32_t* ent_s = reinterpret_cast<int32_t*>(tmem_slot + 4);     // [128] epilogue: entry ids
    float* gate_s = reinterpret_cast<float*>(ent_s + 128);           // [128] epilogue: gates
    uint32_t* sz_tab = reinterpret_cast<uint32_t*>(gate_s + 128);    // [2 groups][128 rows][17] scale|zero

    const int K = PHASE == 0 ? a.H : a.I;
    const int nmb = PHASE == 0 ? a.I / 64 : (a.H + 127) / 128;
    const int nk = K / KCH;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // prologue independent of the predecessor kernels (overlaps their tail under PDL)
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < C::NA; ++b) { mbar_init(&aready[b], 128); mbar_init(&aempty[b], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 128); }
        fence_mbar_init();
        for (int i = 0; i < 4; ++i) tma_prefetch(&maps.xb[i]);
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tmem_a = tmem + 2 * C::NBMAX;          // first TMEM A buffer column
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int n_items = a.n_act[0] * nmb;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int it = 0;
            for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
                const Item w = decode(a, item, nmb);
                const CUtensorMap* amap = PHASE == 0 ? (w.bits == 16 ? &maps.a16_gu : (w.ti ? &maps.ahi_gu : &maps.alo_gu))
                                                     : (w.bits == 16 ? &maps.a16_dn : (w.ti ? &maps.ahi_dn : &maps.alo_dn));
                tma_prefetch(amap);
                const int nb = C::nb(w.bits), ks = C::ks(w.bits);
                const int rawc = 128 * KCH * w.bits / 8;          // raw bytes per chunk (int tiers)
                for (int n0 = 0; n0 < w.m; n0 += nb) {
                    const int rb = box_rows(min(nb, w.m - n0));
                    const CUtensorMap* bmap = &maps.xb[rb == 16 ? 0 : rb == 32 ? 1 : rb == 64 ? 2 : 3];
                    for (int kb0 = 0; kb0 < nk; kb0 += ks, ++it) {
                        const int kc = min(ks, nk - kb0);
                        const int st = it % STAGES, ph = (it / STAGES) & 1;
                        mbar_wait(&empty[st], ph ^ 1);
                        uint8_t* sA = sS + st * STAGE_BYTES;
                        uint8_t* sB = sA + A_BYTES;
                        const uint32_t bytes = kc * rb * 128 + (w.bits == 16 ? A_BYTES : kc * rawc);
                        mbar_arrive_expect_tx(&full[st], bytes);
                        for (int j = 0; j < kc; ++j) {
                            const int kb = kb0 + j;
                            tma_load_2d(sB + j * rb * 128, bmap, &full[st], kb * KCH, w.r0 + n0);
                            if (w.bits == 16) {
                                if (PHASE == 0) {
                                    tma_load_3d(sA, amap, &full[st], kb * KCH, w.mb * 64, w.slot);
                                    tma_load_3d(sA + 64 * 128, amap, &full[st], kb * KCH, a.I + w.mb * 64, w.slot);
                                } else {
                                    tma_load_3d(sA, amap, &full[st], kb * KCH, w.mb * 128, w.slot);
                                }
                            } else {
                                const int kbytes = kb * KCH * w.bits / 8;
                                uint8_t* dst = sA + j * rawc;
                                if (PHASE == 0) {
                                    tma_load_3d(dst, amap, &full[st], kbytes, w.mb * 64, w.slot);
                                    tma_load_3d(dst + rawc / 2, amap, &full[st], kbytes, a.I + w.mb * 64, w.slot);
                                } else {
                                    tma_load_3d(dst, amap, &full[st], kbytes, w.mb * 128, w.slot);
                                }
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (one thread)
        if (lane == 0) {
            int it = 0, ac = 0, cc = 0;
            for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
                const Item w = decode(a, item, nmb);
                const int nb = C::nb(w.bits), ks = C::ks(w.bits);
                for (int n0 = 0; n0 < w.m; n0 += nb, ++cc) {
                    const int rb = box_rows(min(nb, w.m - n0));
                    const uint32_t idesc = idesc_bf16(128, rb);
                    const int buf = cc & 1;
                    mbar_wait(&tempty[buf], ((cc >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem + buf * C::NBMAX;
                    for (int kb0 = 0; kb0 < nk; kb0 += ks, ++it) {
                        const int kc = min(ks, nk - kb0);
                        const int st = it % STAGES, ph = (it / STAGES) & 1;
                        mbar_wait(&full[st], ph);
                        tc_fence_after();
                        const uint32_t sA = smem_u32(sS + st * STAGE_BYTES), sB = sA + A_BYTES;
                        if (w.bits == 16) {
#pragma unroll
                            for (int s = 0; s < KCH / 16; ++s)
                                mma_bf16(d, umma_desc_sw128(sA + 32 * s), umma_desc_sw128(sB + 32 * s), idesc,
                                         (kb0 | s) != 0);
                        } else {
                            for (int j = 0; j < kc; ++j, ++ac) {
                                const int ab = ac % C::NA;
                                mbar_wait(&aready[ab], (ac / C::NA) & 1);
                                tc_fence_after();
                                const uint32_t at = tmem_a + 32 * ab, bj = sB + j * rb * 128;
#pragma unroll
                                for (int s = 0; s < KCH / 16; ++s)
                                    mma_bf16_ts(d, at + 8 * s, umma_desc_sw128(bj + 32 * s), idesc,
                                                ((kb0 + j) | s) != 0);
                                mma_commit(&aempty[ab]);
                            }
                        }
                        mma_commit(&empty[st]);
                    }
                    mma_commit(&tfull[buf]);
                }
            }
        }
    } else if (warp < 10) {
        // ------------------------------------------------ dequant transform: two 4-warp groups take
        // alternate K chunks of the quantised stages; thread = A row = TMEM lane
        const int grp = (warp - 2) >> 2;
        const int qa = warp & 3;
        const int r = 32 * qa + lane;
        const int rows_total = PHASE == 0 ? 2 * a.I : a.H;
        const int mat = PHASE == 0 ? 0 : 2;
        const int G = K / a.g;
        int it = 0, ac = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
            const Item w = decode(a, item, nmb);
            const int nb = C::nb(w.bits), ks = C::ks(w.bits);
            const int mat_row = PHASE == 0 ? (r < 64 ? 0 : a.I) + w.mb * 64 + (r & 63) : w.mb * 128 + r;
            const SlotLayout& L = w.ti ? a.hi : a.lo;
            const uint8_t* slot_base =
                a.layer + (w.ti ? a.hi_base + (int64_t)w.slot * a.hi.bytes : (int64_t)w.slot * a.lo.bytes);
            const uint16_t* scales = reinterpret_cast<const uint16_t*>(slot_base + L.scales_off + mat * L.scales_stride);
            const uint8_t* zeros = slot_base + L.zeros_off + mat * L.zeros_stride;
            const int rawc = 128 * KCH * w.bits / 8, rowb = KCH * w.bits / 8;
            // this row's scales / zeros for the whole item, once (G <= 16: g = 128, K <= 2048), packed
            // as (bf16 scale | bf16(128 + z) << 16); otherwise fetched per chunk
            // thread-private row table in smem (only this thread writes and reads it)
            uint32_t* sz = sz_tab + (grp * 128 + r) * 17;
            const bool sz_reg = G <= 16 && w.bits != 16;
            if (sz_reg) {
                for (int gi = 0; gi < G; ++gi) {
                    uint32_t v = 0x43003f80u;
                    if (mat_row < rows_total)
                        v = (uint32_t)scales[(int64_t)mat_row * G + gi] | ((0x4300u + zeros[(int64_t)mat_row * G + gi]) << 16);
                    sz[gi] = v;
                }
            }
            for (int n0 = 0; n0 < w.m; n0 += nb) {
                for (int kb0 = 0; kb0 < nk; kb0 += ks, ++it) {
                    const int st = it % STAGES, ph = (it / STAGES) & 1;
                    // every transform thread observes every phase of full[] (no phase aliasing)
                    mbar_wait(&full[st], ph);
                    if (w.bits == 16) continue;                   // bf16 stages need no transform
                    const int kc = min(ks, nk - kb0);
                    for (int j = 0; j < kc; ++j, ++ac) {
                        if ((ac & 1) != grp) continue;
                        const int kb = kb0 + j;
                        uint32_t zz[2], ss[2];
#pragma unroll
                        for (int h2 = 0; h2 < 2; ++h2) {           // one or two groups per 64-element chunk
                            const int gi = (kb * KCH + h2 * 32) / a.g;
                            uint32_t v = 0x43003f80u;
                            if (sz_reg) {
                                v = sz[gi];
                            } else if (mat_row < rows_total) {
                                v = (uint32_t)scales[(int64_t)mat_row * G + gi] |
                                    ((0x4300u + zeros[(int64_t)mat_row * G + gi]) << 16);
                            }
                            zz[h2] = (v >> 16) * 0x10001u;
                            ss[h2] = (v & 0xFFFFu) * 0x10001u;
                        }
                        const int ab = ac % C::NA;
                        mbar_wait(&aempty[ab], ((ac / C::NA) & 1) ^ 1);
                        const uint32_t raw_addr = smem_u32(sS + st * STAGE_BYTES + j * rawc + r * rowb);
                        uint32_t wv[KCH / 2];                      // 32 bf16x2 words = 64 elements
                        if (a.dbg == 1) {                          // perf experiment: no dequant
#pragma unroll
                            for (int b = 0; b < 32; ++b) wv[b] = zz[0] ^ b;
                        } else if (w.bits == 4) {
                            uint32_t s0, s1, s2, s3, s4, s5, s6, s7;
                            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3) : "r"(raw_addr));
                            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(s4), "=r"(s5), "=r"(s6), "=r"(s7) : "r"(raw_addr + 16));
                            const uint32_t src[8] = {s0, s1, s2, s3, s4, s5, s6, s7};
#pragma unroll
                            for (int b = 0; b < 32; ++b) {      // pair-interleaved: pair j at bits 4j, 16+4j
                                const uint32_t x = src[b >> 2] >> (4 * (b & 3));
                                wv[b] = bf2_sub_mul((x & 0x000F000Fu) | 0x43004300u, zz[b >> 4], ss[b >> 4]);
                            }
                        } else {
                            uint32_t s0, s1, s2, s3;
                            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3) : "r"(raw_addr));
                            const uint32_t src[4] = {s0, s1, s2, s3};
#pragma unroll
                            for (int b = 0; b < 32; ++b) {      // pair-interleaved: pair j at bits 2j, 16+2j
                                const uint32_t x = src[b >> 3] >> (2 * (b & 7));
                                wv[b] = bf2_sub_mul((x & 0x00030003u) | 0x43004300u, zz[b >> 4], ss[b >> 4]);
                            }
                        }
                        tc_fence_after();
                        if (a.dbg != 2) {                          // dbg 2: perf experiment, no TMEM store
                            tmem_st32(tmem_a + ((uint32_t)(32 * qa) << 16) + 32 * ab, wv);
                            tmem_st_wait();
                        } else if (wv[lane] == 0x12345678u) {
                            a.act[0] = __float2bfloat16_rn(0.0f);
                        }
                        tc_fence_before();
                        mbar_arrive(&aready[ab]);
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------ epilogue (128 threads, warps 10-13)
        const int q = warp & 3;                         // TMEM lane quarter this warp may access
        const int et = threadIdx.x - 320;               // 0..127
        int cc = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
            const Item w = decode(a, item, nmb);
            const int nb = C::nb(w.bits);
            for (int n0 = 0; n0 < w.m; n0 += nb, ++cc) {
                const int buf = cc & 1;
                const int nvalid = min(nb, w.m - n0);
                if (PHASE == 1) {                       // entry ids and gates of this chunk's tokens -> smem
                    for (int i = et; i < nvalid; i += 128) {
                        const int ent = a.perm[w.r0 + n0 + i];
                        ent_s[i] = ent;
                        gate_s[i] = a.gate[ent];
                    }
                }
                mbar_wait(&tfull[buf], (cc >> 1) & 1);
                tc_fence_after();
                named_bar(1, 128);
                for (int col = 0; col < nvalid; col += 32) {
                    uint32_t v[32];
                    tmem_ld32(tmem + buf * C::NBMAX + ((uint32_t)(32 * q) << 16) + col, v);
                    tmem_ld_wait();
                    if (PHASE == 0) {
                        // rows 64-127 (up) -> smem; rows 0-63 (gate) combine: act = silu(g) * u
                        if (q >= 2) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) xch[j * 64 + 32 * (q - 2) + lane] = __uint_as_float(v[j]);
                        }
                        named_bar(1, 128);
                        if (q < 2) {
                            const int f = w.mb * 64 + 32 * q + lane;
#pragma unroll
                            for (int j = 0; j < 32; ++j) {           // fully unrolled: v[] stays in registers
                                if (col + j < nvalid) {
                                    const float gv = __uint_as_float(v[j]);
                                    const float uv = xch[j * 64 + 32 * q + lane];
                                    const float sg = gv / (1.0f + __expf(-gv));
                                    a.act[(size_t)(w.r0 + n0 + col + j) * a.I + f] = __float2bfloat16_rn(sg * uv);
                                }
                            }
                        }
                        named_bar(1, 128);
                    } else {
                        const int h = w.mb * 128 + 32 * q + lane;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {           // fully unrolled: v[] stays in registers
                            if (col + j < nvalid && h < a.H) {
                                const int ent = ent_s[col + j];
                                a.Y[(size_t)ent * a.H + h] = __float2bfloat16_rn(gate_s[col + j] * __uint_as_float(v[j]));
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(&tempty[buf]);
                named_bar(1, 128);                      // ent_s / gate_s / xch reused by the next chunk
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int PHASE, bool DEC>
void launch_one(const GemmMaps& maps, const GemmArgs& a, int items, cudaStream_t st) {
    using C = Cfg<DEC>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gemm<PHASE, DEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        attr = true;
    }
    const int grid = items < DX_NUM_SMS ? items : DX_NUM_SMS;    // persistent: one CTA per SM
    dx_launch(k_gemm<PHASE, DEC>, dim3(grid), dim3(GEMM_THREADS), C::SMEM, st, g_dx_pdl, maps, a);
}

}  // namespace

bool gemm_decode_cfg(int T) { return T <= 64; }

void launch_gemm(int phase, bool dec, const GemmMaps& maps, const GemmArgs& a, int max_items, cudaStream_t st) {
    if (max_items <= 0) return;
    if (phase == 0) {
        if (dec) launch_one<0, true>(maps, a, max_items, st);
        else launch_one<0, false>(maps, a, max_items, st);
    } else {
        if (dec) launch_one<1, true>(maps, a, max_items, st);
        else launch_one<1, false>(maps, a, max_items, st);
    }
}
