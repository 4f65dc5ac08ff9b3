// dx_quant.cuh -- group quantiser device functions (DESIGN.md R-Q1), shared by the standalone
// quantiser kernel (k_quant.cu) and the side-stream demotion kernel (k_ctrl.cu).
//
// Two packings of the codes of a row:
//  * canonical (the standalone dx_quantize API): little-endian along K, element k at bit (k*bits)
//    of its byte stream;
//  * pair-interleaved (PI, the physical layout inside pool slots): 32-bit little-endian words of
//    W = 32/bits consecutive elements, element e of a word at slot e/2 if e is even, W/2 + e/2 if odd.
//    The pair (2j, 2j+1) then sits at bits (bits*j, 16 + bits*j): one shift and one LOP3 produce the
//    two codes in the two bf16 halves of a register (the dequant hot loop).  Exports un-interleave.
#pragma once
#include "dx_common.cuh"

__device__ __forceinline__ int dxq_pi_slot(int e, int W) { return (e & 1) ? (W >> 1) + (e >> 1) : (e >> 1); }

// code of element k of a packed row
__device__ __forceinline__ int dxq_code(const uint8_t* row, int64_t k, int bits, bool pi) {
    const int mask = (1 << bits) - 1;
    if (!pi) {
        const int per = 8 / bits;
        return (row[k / per] >> ((k % per) * bits)) & mask;
    }
    const int W = 32 / bits;
    const uint32_t word = reinterpret_cast<const uint32_t*>(row)[k / W];
    return (word >> (bits * dxq_pi_slot((int)(k % W), W))) & mask;
}

// Fetch the EPL elements of lane `lane` in group (row n, group gi) as fp32 (dequantised exactly when
// the source is quantised: bf16_rn((q - z) * s)).
template <int EPL>
__device__ __forceinline__ void dxq_fetch_group(const void* src, int src_bits, const uint8_t* s_scales,
                                                const uint8_t* s_zeros, int64_t n, int64_t gi, int64_t K,
                                                int g, int lane, float (&w)[EPL], bool pi) {
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
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
            const int q = dxq_code(codes, k0 + i, src_bits, pi);
            w[i] = __bfloat162float(__float2bfloat16_rn(__fmul_rn((float)(q - z), s)));
        }
    }
}

// Quantise one group of g = 32*EPL elements held EPL per lane; writes packed codes of row `row`
// (K elements, `bits` per code, canonical or PI packing), its bf16 scale and u8 zero.  Warp-collective.
template <int EPL>
__device__ __forceinline__ void dxq_quantize_group(const float (&w)[EPL], int bits, int64_t gi, int64_t K,
                                                   int lane, uint8_t* __restrict__ row,
                                                   __nv_bfloat16* __restrict__ scale_out,
                                                   uint8_t* __restrict__ zero_out, bool pi) {
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
    uint32_t qv[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
        float q = __fadd_rn(rintf(__fdiv_rn(w[i], s)), z);
        qv[i] = (uint32_t)fminf(fmaxf(q, 0.0f), qmax);
    }
    const int64_t k0 = gi * g + (int64_t)lane * EPL;
    if (pi) {
        const int W = 32 / bits, LPW = W / EPL;     // lanes sharing one 32-bit word (power of two)
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < EPL; ++i) v |= qv[i] << (bits * dxq_pi_slot((int)((k0 + i) % W), W));
        for (int o = 1; o < LPW; o <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
        if (lane % LPW == 0) reinterpret_cast<uint32_t*>(row)[k0 / W] = v;
    } else {
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < EPL; ++i) v |= qv[i] << (i * bits);
        const int LB = EPL * bits;
        const int64_t bit0 = k0 * bits;
        if (LB >= 8) {
            for (int b = 0; b < LB / 8; ++b) row[bit0 / 8 + b] = (uint8_t)(v >> (8 * b));
        } else {
            const int LPB = 8 / LB;
            uint32_t acc = 0;
            const int base = lane - lane % LPB;
            for (int i = 0; i < LPB; ++i) acc |= __shfl_sync(0xffffffffu, v, base + i) << (i * LB);
            if (lane % LPB == 0) row[bit0 / 8] = (uint8_t)acc;
        }
    }
    if (lane == 0) { *scale_out = sb; *zero_out = (uint8_t)z; }
}
