// dx_quant.cuh -- group quantiser device functions (DESIGN.md R-Q1), shared by the standalone
// quantiser kernel (k_quant.cu) and the side-stream demotion kernel (k_ctrl.cu).
#pragma once
#include "dx_common.cuh"

// Fetch the EPL elements of lane `lane` in group (row n, group gi) as fp32.
template <int EPL>
__device__ __forceinline__ void dxq_fetch_group(const void* src, int src_bits, const uint8_t* s_scales,
                                            const uint8_t* s_zeros, int64_t n, int64_t gi, int64_t K,
                                            int g, int lane, float (&w)[EPL]) {
    const int64_t k0 = gi * g + (int64_t)lane * EPL;
    if (src_bits == 16) {
        const uint16_t* p = reinterpret_cast<const uint16_t*>(src) + n * K + k0;
#pragma unroll
        for (int i = 0; i < EPL; ++i) w[i] = dx_bf2f(p[i]);
    } else {
        const uint8_t* codes = reinterpret_cast<const uint8_t*>(src) + n * (K * src_bits / 8);
        const int64_t G = K / g;
        float s = dx_bf2f(reinterpret_cast<const uint16_t*>(s_scales)[n * G + gi]);
        int z = s_zeros[n * G + gi];
        const int per = 8 / src_bits, mask = (1 << src_bits) - 1;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
            int64_t k = k0 + i;
            int q = (codes[k / per] >> ((k % per) * src_bits)) & mask;
            w[i] = __bfloat162float(__float2bfloat16_rn(__fmul_rn((float)(q - z), s)));
        }
    }
}

// Quantise one group of g = 32*EPL elements held EPL per lane; writes packed codes of row `row`
// (K elements, `bits` per code), its bf16 scale and u8 zero.  Warp-collective.
template <int EPL>
__device__ __forceinline__ void dxq_quantize_group(const float (&w)[EPL], int bits, int64_t gi, int64_t K,
                                                   int lane, uint8_t* __restrict__ row,
                                                   __nv_bfloat16* __restrict__ scale_out,
                                                   uint8_t* __restrict__ zero_out) {
    const int g = 32 * EPL;
    float lo = 0.0f, hi = 0.0f;     // zero always inside the range
#pragma unroll
    for (int i = 0; i < EPL; ++i) { lo = fminf(lo, w[i]); hi = fmaxf(hi, w[i]); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const float qmax = (float)((1 << bits) - 1);
    float s32 = __fdiv_rn(__fsub_rn(hi, lo), qmax);
    if (s32 == 0.0f) s32 = 1.0f;
    const __nv_bfloat16 sb = __float2bfloat16_ru(s32);
    const float s = __bfloat162float(sb);
    float z = rintf(__fdiv_rn(-lo, s));
    z = fminf(fmaxf(z, 0.0f), qmax);
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
        float q = __fadd_rn(rintf(__fdiv_rn(w[i], s)), z);
        q = fminf(fmaxf(q, 0.0f), qmax);
        v |= ((uint32_t)q) << (i * bits);
    }
    const int LB = EPL * bits;
    const int64_t bit0 = (gi * g + (int64_t)lane * EPL) * bits;
    if (LB >= 8) {
        for (int b = 0; b < LB / 8; ++b) row[bit0 / 8 + b] = (uint8_t)(v >> (8 * b));
    } else {
        const int LPB = 8 / LB;
        uint32_t acc = 0;
        const int base = lane - lane % LPB;
        for (int i = 0; i < LPB; ++i) acc |= __shfl_sync(0xffffffffu, v, base + i) << (i * LB);
        if (lane % LPB == 0) row[bit0 / 8] = (uint8_t)acc;
    }
    if (lane == 0) { *scale_out = sb; *zero_out = (uint8_t)z; }
}
