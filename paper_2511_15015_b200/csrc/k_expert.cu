// k_expert.cu -- decode-regime grouped expert FFN over the slot pool (a6, a7, a9).
//   Eq. 1: E_j(x) = W_down (silu(W_gate x) * W_up x), each expert read from its
//   stable slot at its current tier; LOW/HIGH blocks in the formats of R-Q1.
//
// Design (DESIGN.md §5 "decode kernels"): weight streaming with tensor cores, dequantisation in
// registers.  A CTA owns 2 m-tiles of 16 weight rows of one expert and the full K; its 8 warps
// split K.  Each thread loads 16 consecutive K-elements of rows g and g+8 of a tile per 64-K block
// (bf16: 2x16 B, int4: 8 B, int2: 4 B; coalesced along rows), dequantises exactly
// (bf16_rn((q-z)*s) via bf16x2 magic-number conversion, __hsub2/__hmul2) and feeds
// mma.m16n8k16 with a K permutation shared by A and B: logical k-slots {2t,2t+1 | 2t+8,2t+9} of
// step s <-> physical k = 16t+4s+{0,1 | 2,3}, so the x fragments are plain 32 B loads too.
// Partial tiles are reduced across warps through shared memory; fp32 accumulation throughout.
#include "dx_common.cuh"

#define FFN_WARPS 8
#define FFN_KB 64

namespace {

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t bf2_sub_mul(uint32_t v, uint32_t zz, uint32_t ss) {
    __nv_bfloat162 r = __hmul2(__hsub2(*reinterpret_cast<__nv_bfloat162*>(&v),
                                       *reinterpret_cast<__nv_bfloat162*>(&zz)),
                               *reinterpret_cast<__nv_bfloat162*>(&ss));
    return *reinterpret_cast<uint32_t*>(&r);
}

// 16 consecutive weights of one row (this thread's slice of a 64-K block) as 8 bf16x2 words,
// word w = elements (2w, 2w+1).
template <int BITS>
struct RowSlice {
    uint32_t raw[BITS == 16 ? 8 : (BITS == 4 ? 2 : 1)];
    uint32_t zz, ss;   // bf16x2 (128+z, 128+z), (s, s)
};

template <int BITS>
__device__ __forceinline__ void load_slice(RowSlice<BITS>& r, const MatView& mv, int64_t row, int K, int g,
                                           int k0) {
    if constexpr (BITS == 16) {
        const uint4* p = reinterpret_cast<const uint4*>(mv.codes + (row * K + k0) * 2);
        uint4 a = __ldg(p), b = __ldg(p + 1);
        r.raw[0] = a.x; r.raw[1] = a.y; r.raw[2] = a.z; r.raw[3] = a.w;
        r.raw[4] = b.x; r.raw[5] = b.y; r.raw[6] = b.z; r.raw[7] = b.w;
    } else {
        const uint8_t* p = mv.codes + (row * K + k0) * BITS / 8;
        if constexpr (BITS == 4) {
            uint2 a = __ldg(reinterpret_cast<const uint2*>(p));
            r.raw[0] = a.x; r.raw[1] = a.y;
        } else {
            r.raw[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
        }
        const int64_t G = K / g;
        const uint16_t sb = __ldg(reinterpret_cast<const unsigned short*>(mv.scales) + row * G + k0 / g);
        const uint32_t z = __ldg(mv.zeros + row * G + k0 / g);
        const uint32_t zb = __float_as_uint(128.0f + (float)z) >> 16;   // exact in bf16 (<= 8 bits)
        r.zz = zb | (zb << 16);
        r.ss = (uint32_t)sb | ((uint32_t)sb << 16);
    }
}

// bf16x2 word w (elements 2w, 2w+1) of the slice, dequantised exactly.
template <int BITS>
__device__ __forceinline__ uint32_t slice_word(const RowSlice<BITS>& r, int w) {
    if constexpr (BITS == 16) {
        return r.raw[w];
    } else if constexpr (BITS == 4) {
        // pair-interleaved slot packing (dx_quant.cuh): codes (2w, 2w+1) at bits 4j, 16+4j of word w/4
        const uint32_t x = r.raw[w >> 2] >> (4 * (w & 3));
        return bf2_sub_mul((x & 0x000F000Fu) | 0x43004300u, r.zz, r.ss);
    } else {
        const uint32_t x = r.raw[0] >> (2 * w);                         // bits 2w, 16+2w
        return bf2_sub_mul((x & 0x00030003u) | 0x43004300u, r.zz, r.ss);
    }
}

struct TileSrc {
    MatView mv;
    int64_t row0;      // first of 16 rows
};

// Accumulate RT m-tiles x NT n-tiles over this warp's share of K blocks.
// xs: shared bf16 [NT*8][xstride_words*2], padded rows.
template <int BITS, int RT, int NT>
__device__ __forceinline__ void warp_tiles(const TileSrc (&src)[RT], int K, int g, const uint32_t* xs,
                                           int xstride_words, float (&acc)[RT][NT][4]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane >> 2, t = lane & 3;
    const int nb = K / FFN_KB;
    for (int b = warp; b < nb; b += FFN_WARPS) {
        const int k0 = b * FFN_KB + 16 * t;
        RowSlice<BITS> lo[RT], hi[RT];
#pragma unroll
        for (int r = 0; r < RT; ++r) {
            load_slice<BITS>(lo[r], src[r].mv, src[r].row0 + gq, K, g, k0);
            load_slice<BITS>(hi[r], src[r].mv, src[r].row0 + gq + 8, K, g, k0);
        }
        uint32_t bx[NT][8];
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            const uint4* p = reinterpret_cast<const uint4*>(xs + (n * 8 + gq) * xstride_words + k0 / 2);
            uint4 a = p[0], c = p[1];
            bx[n][0] = a.x; bx[n][1] = a.y; bx[n][2] = a.z; bx[n][3] = a.w;
            bx[n][4] = c.x; bx[n][5] = c.y; bx[n][6] = c.z; bx[n][7] = c.w;
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) {
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                uint32_t a[4];
                a[0] = slice_word<BITS>(lo[r], 2 * s);
                a[1] = slice_word<BITS>(hi[r], 2 * s);
                a[2] = slice_word<BITS>(lo[r], 2 * s + 1);
                a[3] = slice_word<BITS>(hi[r], 2 * s + 1);
#pragma unroll
                for (int n = 0; n < NT; ++n) mma_bf16(acc[r][n], a, bx[n][2 * s], bx[n][2 * s + 1]);
            }
        }
    }
}

__device__ __forceinline__ MatView mat_of(const ExpertArgs& a, int e, int m) {
    const int tier = a.tier[e];
    const SlotLayout& L = tier ? a.hi : a.lo;
    const uint8_t* base = a.arena_layer + (tier ? a.hi_base + (int64_t)a.slot[e] * a.hi.bytes
                                                : (int64_t)a.slot[e] * a.lo.bytes);
    MatView v;
    v.bits = L.bits;
    v.codes = base + m * L.codes_stride;
    v.scales = reinterpret_cast<const __nv_bfloat16*>(base + L.scales_off + m * L.scales_stride);
    v.zeros = base + L.zeros_off + m * L.zeros_stride;
    return v;
}

// PHASE 0: gate/up + SwiGLU -> act (permuted rows);  PHASE 1: down + gate scale -> Y (entry rows)
template <int PHASE, int NT>
__global__ void __launch_bounds__(256) k_ffn(ExpertArgs a, const __nv_bfloat16* __restrict__ x,
                                             const float* __restrict__ gate, const int32_t* __restrict__ perm,
                                             const int32_t* __restrict__ off, const int32_t* __restrict__ act_e,
                                             const int32_t* __restrict__ n_act,
                                             __nv_bfloat16* __restrict__ act, __nv_bfloat16* __restrict__ Y) {
    constexpr int RT = 2;
    extern __shared__ __align__(16) uint32_t smem[];
    DX_GRID_WAIT();
    DX_GRID_LAUNCH();
    const int K = PHASE == 0 ? a.H : a.I;
    const int rows_per_item = PHASE == 0 ? 16 : 32;
    const int nrb = (PHASE == 0 ? a.I : a.H) / rows_per_item;
    const int item = blockIdx.x;
    if (item >= n_act[0] * nrb) return;
    const int e = act_e[item / nrb];
    const int rb = item % nrb;
    const int r0 = off[e], m = off[e + 1] - r0;
    const int xstride = K / 2 + 4;                       // words; +16 B pad against bank conflicts
    uint32_t* xs = smem;
    float* red = reinterpret_cast<float*>(smem + NT * 8 * xstride);   // [8 warps][RT][NT][32][4]
    TileSrc src[RT];
    if (PHASE == 0) {
        src[0].mv = mat_of(a, e, 0); src[0].row0 = rb * 16;
        src[1].mv = mat_of(a, e, 1); src[1].row0 = rb * 16;
    } else {
        src[0].mv = mat_of(a, e, 2); src[0].row0 = rb * 32;
        src[1].mv = src[0].mv;       src[1].row0 = rb * 32 + 16;
    }
    const int bits = src[0].mv.bits;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int p0 = 0; p0 < m; p0 += NT * 8) {
        const int mt = min(NT * 8, m - p0);
        __syncthreads();
        // stage x rows of this pass (bf16, padded)
        const int chunks = K / 8;
        for (int i = threadIdx.x; i < NT * 8 * chunks; i += blockDim.x) {
            const int r = i / chunks, c = i % chunks;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (r < mt) {
                const __nv_bfloat16* srow;
                if (PHASE == 0) srow = x + (size_t)(perm[r0 + p0 + r] / a.k) * K;
                else            srow = act + (size_t)(r0 + p0 + r) * K;
                v = *reinterpret_cast<const uint4*>(srow + c * 8);
            }
            *reinterpret_cast<uint4*>(xs + r * xstride + c * 4) = v;
        }
        __syncthreads();
        float acc[RT][NT][4];
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[r][n][q] = 0.0f;
        if (bits == 16)      warp_tiles<16, RT, NT>(src, K, a.g, xs, xstride, acc);
        else if (bits == 4)  warp_tiles<4, RT, NT>(src, K, a.g, xs, xstride, acc);
        else                 warp_tiles<2, RT, NT>(src, K, a.g, xs, xstride, acc);
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
            for (int n = 0; n < NT; ++n)
                *reinterpret_cast<float4*>(red + ((((warp * RT + r) * NT + n) * 32 + lane) * 4)) =
                    make_float4(acc[r][n][0], acc[r][n][1], acc[r][n][2], acc[r][n][3]);
        __syncthreads();
        // reduce over warps: element (r, row, tok) lives at lane = (row%8)*4 + (tok%8)/2,
        // q = (row/8)*2 + tok%2 of n-tile tok/8
        for (int o = threadIdx.x; o < 16 * NT * 8; o += blockDim.x) {
            const int row = o / (NT * 8), tok = o % (NT * 8);
            if (tok >= mt) continue;
            const int n = tok / 8, tt = tok % 8;
            const int ln = (row % 8) * 4 + tt / 2, q = (row / 8) * 2 + (tt % 2);
            float v0 = 0.0f, v1 = 0.0f;
#pragma unroll
            for (int w = 0; w < FFN_WARPS; ++w) {
                v0 += red[(((w * RT + 0) * NT + n) * 32 + ln) * 4 + q];
                v1 += red[(((w * RT + 1) * NT + n) * 32 + ln) * 4 + q];
            }
            if (PHASE == 0) {
                const float sg = v0 / (1.0f + expf(-v0));
                act[(size_t)(r0 + p0 + tok) * a.I + rb * 16 + row] = __float2bfloat16_rn(sg * v1);
            } else {
                const int ent = perm[r0 + p0 + tok];
                const float gt = gate[ent];
                Y[(size_t)ent * a.H + rb * 32 + row] = __float2bfloat16_rn(gt * v0);
                Y[(size_t)ent * a.H + rb * 32 + 16 + row] = __float2bfloat16_rn(gt * v1);
            }
        }
    }
}

template <int PHASE, int NT>
void launch_phase(const ExpertArgs& a, const __nv_bfloat16* x, const float* gate, const RouteWs& ws,
                  int max_items, __nv_bfloat16* act, __nv_bfloat16* Y, cudaStream_t st) {
    const int K = PHASE == 0 ? a.H : a.I;
    const size_t sm = (size_t)NT * 8 * (K / 2 + 4) * 4 + (size_t)FFN_WARPS * 2 * NT * 32 * 4 * 4;
    static unsigned long long attr_mask = 0;
    if (dx_first_on_device(attr_mask)) {
        cudaFuncSetAttribute(k_ffn<PHASE, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    if (max_items <= 0) return;
    dx_launch(k_ffn<PHASE, NT>, dim3(max_items), dim3(256), sm, st, g_dx_pdl, a, x, gate, (const int32_t*)ws.perm,
              (const int32_t*)ws.off, (const int32_t*)ws.act_e, (const int32_t*)ws.n_act, act, Y);
}

}  // namespace

void launch_expert_ffn(const ExpertArgs& a, const __nv_bfloat16* x, const float* gate, const RouteWs& ws,
                       int T, int E, __nv_bfloat16* act, __nv_bfloat16* Y, cudaStream_t st, cudaEvent_t mid) {
    if (T <= 0) return;
    const int max_act = T * a.k < E ? T * a.k : E;
    const int items0 = max_act * (a.I / 16), items1 = max_act * (a.H / 32);
    if (T <= 8) {
        launch_phase<0, 1>(a, x, gate, ws, items0, act, Y, st);
        if (mid) cudaEventRecord(mid, st);
        launch_phase<1, 1>(a, x, gate, ws, items1, act, Y, st);
    } else {
        launch_phase<0, 2>(a, x, gate, ws, items0, act, Y, st);
        if (mid) cudaEventRecord(mid, st);
        launch_phase<1, 2>(a, x, gate, ws, items1, act, Y, st);
    }
}
