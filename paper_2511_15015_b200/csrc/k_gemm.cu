// k_gemm.cu -- tcgen05 grouped expert GEMMs over the slot pool (a6 gate/up + SwiGLU, a7 down + gate
// scaling), one kernel per phase, every touched expert at its stable tier.
//   Eq. 1: E_j(x) = W_down (silu(W_gate x) * W_up x).
//
// Swap-AB: the weights are the M = 128 operand (A, K-major in shared memory, 128 B swizzle), the
// tokens of one expert are N (B, K-major), the accumulator D[128 x BN] fp32 lives in TMEM.
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + single-thread MMA issuer,
// warps 2-5 = dequant transform (quantised tiers: raw codes TMA'd to smem -> bf16 SW128 A tile,
// exactly bf16_rn((q-z)s), R-Q1) and epilogue (tcgen05.ld -> SwiGLU / gate scale -> global).
// bf16 tiers are TMA'd straight into the swizzled A tile.  A 3-8 stage mbarrier ring overlaps TMA,
// dequant and MMA.  Gate/up tiles interleave 16 gate and 16 up rows per 32-lane TMEM quarter so the
// SwiGLU pairs meet in one warp (shfl_xor 16).
#include "dx_common.cuh"
#include "dx_sm100.cuh"

using namespace sm100;

namespace {

constexpr int GEMM_THREADS = 192;
constexpr int KCH = 64;                  // K elements per stage (128 B of bf16)

template <int BN>
struct GemmCfg {
    static constexpr int A_BYTES = 128 * 128;
    static constexpr int B_BYTES = BN * 128;
    static constexpr int RAW_BYTES = 128 * 32;        // int4 worst case
    static constexpr int STAGE = A_BYTES + B_BYTES + RAW_BYTES;
    static constexpr int STAGES = (200 * 1024) / STAGE > 8 ? 8 : (200 * 1024) / STAGE;
    static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
    static constexpr int SMEM = 1024 + STAGES * STAGE + 1024;
};

__device__ __forceinline__ uint32_t bf2_sub_mul(uint32_t v, uint32_t zz, uint32_t ss) {
    __nv_bfloat162 r = __hmul2(__hsub2(*reinterpret_cast<__nv_bfloat162*>(&v), *reinterpret_cast<__nv_bfloat162*>(&zz)),
                               *reinterpret_cast<__nv_bfloat162*>(&ss));
    return *reinterpret_cast<uint32_t*>(&r);
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
    uint64_t* tfull = bars + 3 * C::STAGES;               // accumulator ready
    uint64_t* tempty = tfull + 1;                         // accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

    const int K = PHASE == 0 ? a.H : a.I;
    const int nmb = PHASE == 0 ? a.I / 64 : (a.H + 127) / 128;
    const int item = blockIdx.x;
    if (item >= a.n_act[0] * nmb) return;
    const int e = a.act_e[item / nmb];
    const int mb = item % nmb;
    const int r0 = a.off[e], m = a.off[e + 1] - r0;
    const int ti = a.tier[e], slot = a.slot[e];
    const int bits = ti ? a.hi.bits : a.lo.bits;
    const CUtensorMap* amap = PHASE == 0 ? (bits == 16 ? &maps.a16_gu : (ti ? &maps.ahi_gu : &maps.alo_gu))
                                         : (bits == 16 ? &maps.a16_dn : (ti ? &maps.ahi_dn : &maps.alo_dn));
    const int nk = K / KCH;
    const int nchunk = (m + BN - 1) / BN;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&aready[s], 128); mbar_init(&empty[s], 1); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 128);
        fence_mbar_init();
        tma_prefetch(amap);
        tma_prefetch(&maps.xb);
    }
    if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            const int raw_bytes = 128 * KCH * bits / 8;
            int it = 0;
            for (int c = 0; c < nchunk; ++c) {
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % C::STAGES, ph = (it / C::STAGES) & 1;
                    mbar_wait(&empty[st], ph ^ 1);
                    const uint32_t bytes = C::B_BYTES + (bits == 16 ? C::A_BYTES : raw_bytes);
                    mbar_arrive_expect_tx(&full[st], bytes);
                    tma_load_2d(sB + st * C::B_BYTES, &maps.xb, &full[st], kb * KCH, r0 + c * BN);
                    if (bits == 16) {
                        if (PHASE == 0) {
                            for (int j = 0; j < 8; ++j) {        // 16 gate / 16 up rows per TMEM quarter
                                const int q = j >> 1, part = j & 1;
                                tma_load_3d(sA + st * C::A_BYTES + (32 * q + 16 * part) * 128, amap, &full[st],
                                            kb * KCH, (part ? a.I : 0) + mb * 64 + 16 * q, slot);
                            }
                        } else {
                            tma_load_3d(sA + st * C::A_BYTES, amap, &full[st], kb * KCH, mb * 128, slot);
                        }
                    } else {
                        const int kbytes = kb * KCH * bits / 8;
                        if (PHASE == 0) {
                            tma_load_3d(sR + st * C::RAW_BYTES, amap, &full[st], kbytes, mb * 64, slot);
                            tma_load_3d(sR + st * C::RAW_BYTES + 64 * (KCH * bits / 8), amap, &full[st], kbytes,
                                        a.I + mb * 64, slot);
                        } else {
                            tma_load_3d(sR + st * C::RAW_BYTES, amap, &full[st], kbytes, mb * 128, slot);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(128, BN);
            int it = 0;
            for (int c = 0; c < nchunk; ++c) {
                mbar_wait(tempty, (c & 1) ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % C::STAGES, ph = (it / C::STAGES) & 1;
                    mbar_wait(bits == 16 ? &full[st] : &aready[st], ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + st * C::A_BYTES), b0 = smem_u32(sB + st * C::B_BYTES);
#pragma unroll
                    for (int s = 0; s < KCH / 16; ++s)
                        mma_bf16(tmem, umma_desc_sw128(a0 + 32 * s), umma_desc_sw128(b0 + 32 * s), idesc,
                                 (kb | s) != 0);
                    mma_commit(&empty[st]);
                }
                mma_commit(tfull);
            }
        }
    } else {
        // ------------------------------------------------ transform + epilogue (128 threads)
        const int r = threadIdx.x - 64;                 // A tile row handled by this thread (transform)
        const int q = warp & 3;                         // TMEM lane quarter of this warp (epilogue)
        int raw_row, mat_row;
        if (PHASE == 0) {
            const int qq = r >> 5, i = r & 31;
            raw_row = i < 16 ? 16 * qq + i : 64 + 16 * qq + i - 16;
            mat_row = (i < 16 ? 0 : a.I) + mb * 64 + 16 * qq + (i & 15);
        } else {
            raw_row = r;
            mat_row = mb * 128 + r;
        }
        const int rows_total = PHASE == 0 ? 2 * a.I : a.H;
        const SlotLayout& L = ti ? a.hi : a.lo;
        const uint8_t* slot_base = a.layer + (ti ? a.hi_base + (int64_t)slot * a.hi.bytes : (int64_t)slot * a.lo.bytes);
        const int mat = PHASE == 0 ? 0 : 2;
        const uint16_t* scales = reinterpret_cast<const uint16_t*>(slot_base + L.scales_off + mat * L.scales_stride);
        const uint8_t* zeros = slot_base + L.zeros_off + mat * L.zeros_stride;
        const int G = K / a.g;
        int it = 0;
        for (int c = 0; c < nchunk; ++c) {
            if (bits != 16) {
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % C::STAGES, ph = (it / C::STAGES) & 1;
                    mbar_wait(&full[st], ph);
                    // one or two quantisation groups per 64-element chunk (g = 128/64 or 32)
                    uint32_t zz[2] = {0x43004300u, 0x43004300u}, ss[2] = {0x3f803f80u, 0x3f803f80u};
                    if (mat_row < rows_total) {
#pragma unroll
                        for (int h2 = 0; h2 < 2; ++h2) {
                            const int gi = (kb * KCH + h2 * 32) / a.g;
                            const uint32_t sb = scales[(int64_t)mat_row * G + gi];
                            const uint32_t z = zeros[(int64_t)mat_row * G + gi];
                            const uint32_t zb = __float_as_uint(128.0f + (float)z) >> 16;
                            zz[h2] = zb | (zb << 16);
                            ss[h2] = sb | (sb << 16);
                        }
                    }
                    const uint8_t* raw = sR + st * C::RAW_BYTES + raw_row * (KCH * bits / 8);
                    uint8_t* arow = sA + st * C::A_BYTES + (r >> 3) * 1024 + (r & 7) * 128;
                    uint32_t w[KCH / 2];                 // 32 bf16x2 words = 64 elements
                    if (bits == 4) {
                        const uint4 v0 = *reinterpret_cast<const uint4*>(raw);
                        const uint4 v1 = *reinterpret_cast<const uint4*>(raw + 16);
                        const uint32_t src[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                        for (int b = 0; b < 32; ++b) {
                            const uint32_t x = src[b >> 2] >> (8 * (b & 3));
                            w[b] = bf2_sub_mul((x & 0xFu) | ((x & 0xF0u) << 12) | 0x43004300u, zz[b >> 4], ss[b >> 4]);
                        }
                    } else {
                        const uint4 v0 = *reinterpret_cast<const uint4*>(raw);
                        const uint32_t src[4] = {v0.x, v0.y, v0.z, v0.w};
#pragma unroll
                        for (int b = 0; b < 32; ++b) {
                            const uint32_t x = src[b >> 3] >> (4 * (b & 7));
                            w[b] = bf2_sub_mul((x & 0x3u) | ((x & 0xCu) << 14) | 0x43004300u, zz[b >> 4], ss[b >> 4]);
                        }
                    }
#pragma unroll
                    for (int ch = 0; ch < 8; ++ch)
                        *reinterpret_cast<uint4*>(arow + ((ch ^ (r & 7)) << 4)) =
                            make_uint4(w[4 * ch], w[4 * ch + 1], w[4 * ch + 2], w[4 * ch + 3]);
                    fence_proxy_async_smem();
                    mbar_arrive(&aready[st]);
                }
            }
            // epilogue of chunk c
            mbar_wait(tfull, c & 1);
            tc_fence_after();
            const int n0 = c * BN;
            const int nvalid = min(BN, m - n0);
            for (int col = 0; col < nvalid; col += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + col, v);
                tmem_ld_wait();
                if (PHASE == 0) {
                    const int f = mb * 64 + 16 * q + (lane & 15);
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float gv = __uint_as_float(v[j]);
                        const float uv = __shfl_xor_sync(0xffffffffu, gv, 16);
                        if (lane < 16 && col + j < nvalid) {
                            const float sg = gv / (1.0f + expf(-gv));
                            a.act[(size_t)(r0 + n0 + col + j) * a.I + f] = __float2bfloat16_rn(sg * uv);
                        }
                    }
                } else {
                    const int h = mb * 128 + 32 * q + lane;
#pragma unroll 4
                    for (int j = 0; j < 32; ++j) {
                        if (col + j < nvalid && h < a.H) {
                            const int ent = a.perm[r0 + n0 + col + j];
                            a.Y[(size_t)ent * a.H + h] = __float2bfloat16_rn(a.gate[ent] * __uint_as_float(v[j]));
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tempty);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

// x rows in permuted order: Xp[pos] = x[perm[pos] / k] (B operand of the gate/up GEMM)
__global__ void k_gather(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ perm, int k, int H,
                         __nv_bfloat16* __restrict__ Xp) {
    const int pos = blockIdx.x;
    const int t = perm[pos] / k;
    for (int h = threadIdx.x * 8; h < H; h += blockDim.x * 8)
        *reinterpret_cast<uint4*>(Xp + (size_t)pos * H + h) = *reinterpret_cast<const uint4*>(x + (size_t)t * H + h);
}

template <int PHASE, int BN>
void launch_one(const GemmMaps& maps, const GemmArgs& a, int items, cudaStream_t st) {
    using C = GemmCfg<BN>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gemm<PHASE, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        attr = true;
    }
    k_gemm<PHASE, BN><<<items, GEMM_THREADS, C::SMEM, st>>>(maps, a);
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
    int bn = 32;
    while (bn < T && bn < 256) bn *= 2;
    return bn;
}

void launch_gather(const __nv_bfloat16* x, const int32_t* perm, int rows, int k, int H, __nv_bfloat16* Xp,
                   cudaStream_t st) {
    if (rows <= 0) return;
    int thr = H / 8 < 256 ? H / 8 : 256;
    k_gather<<<rows, thr, 0, st>>>(x, perm, k, H, Xp);
}

void launch_gemm(int phase, int bn, const GemmMaps& maps, const GemmArgs& a, int max_items, cudaStream_t st) {
    if (max_items <= 0) return;
    if (phase == 0) launch_bn<0>(bn, maps, a, max_items, st);
    else launch_bn<1>(bn, maps, a, max_items, st);
}
