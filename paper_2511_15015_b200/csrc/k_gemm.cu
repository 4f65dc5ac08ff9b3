// k_gemm.cu -- tcgen05 grouped expert GEMMs over the slot pool (a6 gate/up + SwiGLU, a7 down + gate
// scaling), one persistent kernel per phase, every touched expert at its stable tier.
//   Eq. 1: E_j(x) = W_down (silu(W_gate x) * W_up x).
//
// Swap-AB: the weights are the M = 128 operand (A, K-major in shared memory, 128 B swizzle), the
// tokens of one expert are N (B, K-major), the accumulator D[128 x BN] fp32 lives in TMEM (two
// buffers, so the epilogue of one work item overlaps the MMAs of the next).
// Persistent CTAs (one per SM) walk the work items (expert, 128-row block) round-robin.
// Warp roles (448 threads): warp 0 = TMA producer, warp 1 = TMEM owner + single-thread MMA issuer,
// warps 2-9 = dequant transform in two groups taking alternate stages (quantised tiers: raw codes
// TMA'd to smem, dequantised exactly to bf16_rn((q-z)s) (R-Q1) and written straight into TMEM as the
// A operand, lane = weight row), warps 10-13 = epilogue (tcgen05.ld -> SwiGLU / gate scale -> global),
// so the epilogue of one item overlaps the mainloop of the next.
// bf16 tiers are TMA'd straight into the swizzled A tile.  An mbarrier ring of 3-8 stages overlaps
// TMA, dequant and MMA.  Gate/up tiles interleave 16 gate and 16 up rows per 32-lane TMEM quarter so
// the SwiGLU pairs meet in one warp (shfl_xor 16).
#include "dx_common.cuh"
#include "dx_sm100.cuh"

using namespace sm100;

namespace {

constexpr int GEMM_THREADS = 448;        // producer, MMA, 2 x 4 transform warps, 4 epilogue warps
constexpr int KCH = 64;                  // K elements per stage (128 B of bf16)

template <int BN>
struct GemmCfg {
    static constexpr int A_BYTES = 128 * 128;
    static constexpr int B_BYTES = BN * 128;
    static constexpr int RAW_BYTES = 128 * 32;        // int4 worst case
    static constexpr int STAGE = A_BYTES + B_BYTES + RAW_BYTES;
    static constexpr int STAGES = (200 * 1024) / STAGE > 8 ? 8 : (200 * 1024) / STAGE;
    // TMEM: ACC_BUFS accumulators of BN columns, then one 32-column A buffer per stage for the
    // quantised tiers (dequantised bf16 A written straight into tensor memory: lane = weight row)
    static constexpr int ACC_BUFS = BN <= 128 ? 2 : 1;
    static constexpr int A_COL0 = ACC_BUFS * BN;
    static constexpr int TMEM_COLS = 512;
    static_assert(A_COL0 + STAGES * 32 <= TMEM_COLS, "TMEM budget");
    static constexpr int SMEM = 1024 + STAGES * STAGE + 1024 + 8 * BN;
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
template <int PHASE>
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

template <int PHASE, int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1) k_gemm(const __grid_constant__ GemmMaps maps, GemmArgs a) {
    using C = GemmCfg<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;                                   // [STAGES][16 KB]
    uint8_t* sB = sA + C::STAGES * C::A_BYTES;            // [STAGES][BN*128]
    uint8_t* sR = sB + C::STAGES * C::B_BYTES;            // [STAGES][4 KB] raw codes
    uint64_t* bars = reinterpret_cast<uint64_t*>(sR + C::STAGES * C::RAW_BYTES);
    uint64_t* full = bars;                                // TMA landed (A or raw, and B)
    uint64_t* aready = bars + C::STAGES;                  // transform wrote A
    uint64_t* empty = bars + 2 * C::STAGES;               // MMA finished with the stage
    uint64_t* tfull = bars + 3 * C::STAGES;               // [2] accumulator ready
    uint64_t* tempty = tfull + 2;                         // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int32_t* ent_s = reinterpret_cast<int32_t*>(tmem_slot + 4);     // [BN] epilogue: entry ids
    float* gate_s = reinterpret_cast<float*>(ent_s + BN);            // [BN] epilogue: gates

    const int K = PHASE == 0 ? a.H : a.I;
    const int nmb = PHASE == 0 ? a.I / 64 : (a.H + 127) / 128;
    const int nk = K / KCH;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // prologue independent of the predecessor kernels (overlaps their tail under PDL)
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&aready[s], 128); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 128); }
        fence_mbar_init();
        tma_prefetch(&maps.xb);
    }
    if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int n_items = a.n_act[0] * nmb;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            int it = 0;
            for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
                const Item w = decode<PHASE>(a, item, nmb);
                const CUtensorMap* amap = PHASE == 0 ? (w.bits == 16 ? &maps.a16_gu : (w.ti ? &maps.ahi_gu : &maps.alo_gu))
                                                     : (w.bits == 16 ? &maps.a16_dn : (w.ti ? &maps.ahi_dn : &maps.alo_dn));
                const int raw_bytes = 128 * KCH * w.bits / 8;
                const int nchunk = (w.m + BN - 1) / BN;
                for (int c = 0; c < nchunk; ++c) {
                    for (int kb = 0; kb < nk; ++kb, ++it) {
                        const int st = it % C::STAGES, ph = (it / C::STAGES) & 1;
                        mbar_wait(&empty[st], ph ^ 1);
                        const uint32_t bytes = C::B_BYTES + (w.bits == 16 ? C::A_BYTES : raw_bytes);
                        mbar_arrive_expect_tx(&full[st], bytes);
                        tma_load_2d(sB + st * C::B_BYTES, &maps.xb, &full[st], kb * KCH, w.r0 + c * BN);
                        if (w.bits == 16) {
                            if (PHASE == 0) {
                                for (int j = 0; j < 8; ++j) {        // 16 gate / 16 up rows per TMEM quarter
                                    const int q = j >> 1, part = j & 1;
                                    tma_load_3d(sA + st * C::A_BYTES + (32 * q + 16 * part) * 128, amap, &full[st],
                                                kb * KCH, (part ? a.I : 0) + w.mb * 64 + 16 * q, w.slot);
                                }
                            } else {
                                tma_load_3d(sA + st * C::A_BYTES, amap, &full[st], kb * KCH, w.mb * 128, w.slot);
                            }
                        } else {
                            const int kbytes = kb * KCH * w.bits / 8;
                            if (PHASE == 0) {
                                tma_load_3d(sR + st * C::RAW_BYTES, amap, &full[st], kbytes, w.mb * 64, w.slot);
                                tma_load_3d(sR + st * C::RAW_BYTES + 64 * (KCH * w.bits / 8), amap, &full[st], kbytes,
                                            a.I + w.mb * 64, w.slot);
                            } else {
                                tma_load_3d(sR + st * C::RAW_BYTES, amap, &full[st], kbytes, w.mb * 128, w.slot);
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(128, BN);
            int it = 0, cc = 0;
            for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
                const Item w = decode<PHASE>(a, item, nmb);
                const int nchunk = (w.m + BN - 1) / BN;
                for (int c = 0; c < nchunk; ++c, ++cc) {
                    const int buf = cc % C::ACC_BUFS;
                    mbar_wait(&tempty[buf], ((cc / C::ACC_BUFS) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem + buf * BN;
                    for (int kb = 0; kb < nk; ++kb, ++it) {
                        const int st = it % C::STAGES, ph = (it / C::STAGES) & 1;
                        mbar_wait(&aready[st], ph);          // every stage use: transform warps arrive
                        tc_fence_after();
                        const uint32_t b0 = smem_u32(sB + st * C::B_BYTES);
                        if (w.bits == 16) {                  // A: bf16 tile TMA'd into smem (SW128)
                            const uint32_t a0 = smem_u32(sA + st * C::A_BYTES);
#pragma unroll
                            for (int s = 0; s < KCH / 16; ++s)
                                mma_bf16(d, umma_desc_sw128(a0 + 32 * s), umma_desc_sw128(b0 + 32 * s), idesc,
                                         (kb | s) != 0);
                        } else {                             // A: dequantised into TMEM by the transform warps
                            const uint32_t at = tmem + C::A_COL0 + 32 * st;
#pragma unroll
                            for (int s = 0; s < KCH / 16; ++s)
                                mma_bf16_ts(d, at + 8 * s, umma_desc_sw128(b0 + 32 * s), idesc, (kb | s) != 0);
                        }
                        mma_commit(&empty[st]);
                    }
                    mma_commit(&tfull[buf]);
                }
            }
        }
    } else if (warp < 10) {
        // ------------------------------------------------ dequant transform: two groups of 4 warps
        // (warps 2-5, 6-9) take alternate stage uses, so two stages are dequantised concurrently
        const int grp = (warp - 2) >> 2;
        const int qa = warp & 3;                        // TMEM lane quarter this warp may write
        const int r = 32 * qa + lane;                   // A tile row (= TMEM lane) handled by this thread
        const int rows_total = PHASE == 0 ? 2 * a.I : a.H;
        const int mat = PHASE == 0 ? 0 : 2;
        const int G = K / a.g;
        int it = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
            const Item w = decode<PHASE>(a, item, nmb);
            int raw_row, mat_row;
            if (PHASE == 0) {
                const int qq = r >> 5, i = r & 31;
                raw_row = i < 16 ? 16 * qq + i : 64 + 16 * qq + i - 16;
                mat_row = (i < 16 ? 0 : a.I) + w.mb * 64 + 16 * qq + (i & 15);
            } else {
                raw_row = r;
                mat_row = w.mb * 128 + r;
            }
            const SlotLayout& L = w.ti ? a.hi : a.lo;
            const uint8_t* slot_base =
                a.layer + (w.ti ? a.hi_base + (int64_t)w.slot * a.hi.bytes : (int64_t)w.slot * a.lo.bytes);
            const uint16_t* scales = reinterpret_cast<const uint16_t*>(slot_base + L.scales_off + mat * L.scales_stride);
            const uint8_t* zeros = slot_base + L.zeros_off + mat * L.zeros_stride;
            const int nchunk = (w.m + BN - 1) / BN;
            for (int c = 0; c < nchunk; ++c) {
                if (w.bits == 16) {
                    // bf16 tier: A arrived by TMA; still consume the stage so that aready[] completes
                    // exactly once per stage use for every tier (keeps all phases in lock-step)
                    for (int kb = 0; kb < nk; ++kb, ++it) {
                        if ((it & 1) != grp) continue;
                        const int st = it % C::STAGES, ph = (it / C::STAGES) & 1;
                        mbar_wait(&full[st], ph);
                        mbar_arrive(&aready[st]);
                    }
                } else {
                    for (int kb = 0; kb < nk; ++kb, ++it) {
                        if ((it & 1) != grp) continue;
                        const int st = it % C::STAGES, ph = (it / C::STAGES) & 1;
                        // scales/zeros first (global, independent of the stage) to overlap the wait
                        uint32_t zz[2] = {0x43004300u, 0x43004300u}, ss[2] = {0x3f803f80u, 0x3f803f80u};
                        if (mat_row < rows_total) {
#pragma unroll
                            for (int h2 = 0; h2 < 2; ++h2) {       // one or two groups per 64-element chunk
                                const int gi = (kb * KCH + h2 * 32) / a.g;
                                const uint32_t sb = scales[(int64_t)mat_row * G + gi];
                                const uint32_t z = zeros[(int64_t)mat_row * G + gi];
                                const uint32_t zb = __float_as_uint(128.0f + (float)z) >> 16;
                                zz[h2] = zb | (zb << 16);
                                ss[h2] = sb | (sb << 16);
                            }
                        }
                        mbar_wait(&full[st], ph);
                        const uint8_t* raw = sR + st * C::RAW_BYTES + raw_row * (KCH * w.bits / 8);
                        uint32_t wv[KCH / 2];                 // 32 bf16x2 words = 64 elements
                        if (w.bits == 4) {
                            const uint4 v0 = *reinterpret_cast<const uint4*>(raw);
                            const uint4 v1 = *reinterpret_cast<const uint4*>(raw + 16);
                            const uint32_t src[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                            for (int b = 0; b < 32; ++b) {
                                const uint32_t x = src[b >> 2] >> (8 * (b & 3));
                                wv[b] = bf2_sub_mul((x & 0xFu) | ((x & 0xF0u) << 12) | 0x43004300u, zz[b >> 4], ss[b >> 4]);
                            }
                        } else {
                            const uint4 v0 = *reinterpret_cast<const uint4*>(raw);
                            const uint32_t src[4] = {v0.x, v0.y, v0.z, v0.w};
#pragma unroll
                            for (int b = 0; b < 32; ++b) {
                                const uint32_t x = src[b >> 3] >> (4 * (b & 7));
                                wv[b] = bf2_sub_mul((x & 0x3u) | ((x & 0xCu) << 14) | 0x43004300u, zz[b >> 4], ss[b >> 4]);
                            }
                        }
                        // row r of the A tile -> TMEM lane r, columns [A_COL0 + 32 st, +32)
                        tmem_st32(tmem + ((uint32_t)(32 * qa) << 16) + C::A_COL0 + 32 * st, wv);
                        tmem_st_wait();
                        tc_fence_before();
                        mbar_arrive(&aready[st]);
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
            const Item w = decode<PHASE>(a, item, nmb);
            const int nchunk = (w.m + BN - 1) / BN;
            for (int c = 0; c < nchunk; ++c, ++cc) {
                const int buf = cc % C::ACC_BUFS;
                const int n0 = c * BN;
                const int nvalid = min(BN, w.m - n0);
                if (PHASE == 1) {                       // entry ids and gates of this chunk's tokens -> smem
                    for (int i = et; i < nvalid; i += 128) {
                        const int ent = a.perm[w.r0 + n0 + i];
                        ent_s[i] = ent;
                        gate_s[i] = a.gate[ent];
                    }
                    named_bar(1, 128);
                }
                mbar_wait(&tfull[buf], (cc / C::ACC_BUFS) & 1);
                tc_fence_after();
                for (int col = 0; col < nvalid; col += 32) {
                    uint32_t v[32];
                    tmem_ld32(tmem + buf * BN + ((uint32_t)(32 * q) << 16) + col, v);
                    tmem_ld_wait();
                    if (PHASE == 0) {
                        const int f = w.mb * 64 + 16 * q + (lane & 15);
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float gv = __uint_as_float(v[j]);
                            const float uv = __shfl_xor_sync(0xffffffffu, gv, 16);
                            if (lane < 16 && col + j < nvalid) {
                                const float sg = gv / (1.0f + expf(-gv));
                                a.act[(size_t)(w.r0 + n0 + col + j) * a.I + f] = __float2bfloat16_rn(sg * uv);
                            }
                        }
                    } else {
                        const int h = w.mb * 128 + 32 * q + lane;
#pragma unroll 8
                        for (int j = 0; j < 32; ++j) {
                            if (col + j < nvalid && h < a.H) {
                                const int ent = ent_s[col + j];
                                a.Y[(size_t)ent * a.H + h] = __float2bfloat16_rn(gate_s[col + j] * __uint_as_float(v[j]));
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(&tempty[buf]);
                if (PHASE == 1) named_bar(1, 128);      // ent_s / gate_s reused by the next chunk
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

template <int PHASE, int BN>
void launch_one(const GemmMaps& maps, const GemmArgs& a, int items, cudaStream_t st) {
    using C = GemmCfg<BN>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gemm<PHASE, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        attr = true;
    }
    const int grid = items < DX_NUM_SMS ? items : DX_NUM_SMS;    // persistent: one CTA per SM
    dx_launch(k_gemm<PHASE, BN>, dim3(grid), dim3(GEMM_THREADS), C::SMEM, st, g_dx_pdl, maps, a);
}

template <int PHASE>
void launch_bn(int bn, const GemmMaps& maps, const GemmArgs& a, int items, cudaStream_t st) {
    switch (bn) {
        case 32: launch_one<PHASE, 32>(maps, a, items, st); break;
        case 64: launch_one<PHASE, 64>(maps, a, items, st); break;
        case 128: launch_one<PHASE, 128>(maps, a, items, st); break;
        default: launch_one<PHASE, 256>(maps, a, items, st); break;
    }
}

}  // namespace

int gemm_bn_for(int T) {
    // N tile: the whole expert in one chunk for decode; 128 (two TMEM accumulators, so the epilogue
    // of one chunk overlaps the MMAs of the next) for prefill
    int bn = 32;
    while (bn < T && bn < 128) bn *= 2;
    return bn;
}

void launch_gemm(int phase, int bn, const GemmMaps& maps, const GemmArgs& a, int max_items, cudaStream_t st) {
    if (max_items <= 0) return;
    if (phase == 0) launch_bn<0>(bn, maps, a, max_items, st);
    else launch_bn<1>(bn, maps, a, max_items, st);
}
