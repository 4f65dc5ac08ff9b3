// k_quant.cu -- on-device group quantiser / dequantiser (K8), DESIGN.md R-Q1.
// Used at pool creation (LOW images, and HIGH images when HIGH is quantised) and by demotion on
// the side stream ("Demotion mirrors this process in reverse").
// Bit-exactness: every arithmetic step is an explicitly IEEE-rounded intrinsic (__fdiv_rn,
// __fsub_rn, __fmul_rn, rintf, __float2bfloat16_ru/_rn); nothing can be contracted.
// Slots use the pair-interleaved code packing (dx_quant.cuh); the standalone API is canonical.
#include "dx_quant.cuh"

namespace {

// One warp per group of g = 32*EPL elements.  src_pi / dst_pi: packing of quantised source / output.
template <int EPL>
__global__ void __launch_bounds__(256) k_quantize(const void* __restrict__ src, int src_bits,
                                                  const uint8_t* __restrict__ s_scales,
                                                  const uint8_t* __restrict__ s_zeros, int64_t N,
                                                  int64_t K, int bits, uint8_t* __restrict__ codes,
                                                  __nv_bfloat16* __restrict__ scales,
                                                  uint8_t* __restrict__ zeros, int src_pi, int dst_pi) {
    const int g = 32 * EPL;
    const int lane = threadIdx.x & 31;
    const int64_t G = K / g;
    const int64_t grp = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (grp >= N * G) return;
    const int64_t n = grp / G, gi = grp % G;
    float w[EPL];
    dxq_fetch_group<EPL>(src, src_bits, s_scales, s_zeros, n, gi, K, g, lane, w, src_pi != 0);
    dxq_quantize_group<EPL>(w, bits, gi, K, lane, codes + n * (K * bits / 8), scales + n * G + gi,
                            zeros + n * G + gi, dst_pi != 0);
}

// 8 outputs per thread (canonical packing).
__global__ void k_dequantize(const uint8_t* __restrict__ codes, const __nv_bfloat16* __restrict__ scales,
                             const uint8_t* __restrict__ zeros, int64_t N, int64_t K, int g, int bits,
                             __nv_bfloat16* __restrict__ out) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c * 8 >= N * K) return;
    const int64_t n = (c * 8) / K, k0 = (c * 8) % K;
    const int64_t G = K / g;
    const float s = __bfloat162float(scales[n * G + k0 / g]);
    const int z = zeros[n * G + k0 / g];
    const uint8_t* row = codes + n * (K * bits / 8);
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int q = dxq_code(row, k0 + i, bits, false);
        o[i] = __float2bfloat16_rn(__fmul_rn((float)(q - z), s));
    }
    *reinterpret_cast<uint4*>(out + n * K + k0) = *reinterpret_cast<const uint4*>(o);
}

void quantize_impl(const void* src, int src_bits, const uint8_t* src_scales, const uint8_t* src_zeros, int64_t N,
                   int64_t K, int g, int bits, uint8_t* codes, __nv_bfloat16* scales, uint8_t* zeros, int src_pi,
                   int dst_pi, cudaStream_t st) {
    const int64_t groups = N * (K / g);
    const int wpb = 8;
    const unsigned blocks = (unsigned)((groups + wpb - 1) / wpb);
    if (blocks == 0) return;
#define DX_QARGS src, src_bits, src_scales, src_zeros, N, K, bits, codes, scales, zeros, src_pi, dst_pi
    switch (g) {
        case 32: k_quantize<1><<<blocks, wpb * 32, 0, st>>>(DX_QARGS); break;
        case 64: k_quantize<2><<<blocks, wpb * 32, 0, st>>>(DX_QARGS); break;
        default: k_quantize<4><<<blocks, wpb * 32, 0, st>>>(DX_QARGS); break;
    }
#undef DX_QARGS
}

}  // namespace

void launch_quantize(const void* src, int src_bits, const uint8_t* src_scales, const uint8_t* src_zeros,
                     int64_t N, int64_t K, int g, int bits, uint8_t* codes, __nv_bfloat16* scales,
                     uint8_t* zeros, cudaStream_t st) {
    quantize_impl(src, src_bits, src_scales, src_zeros, N, K, g, bits, codes, scales, zeros, 0, 0, st);
}

void launch_dequantize(const uint8_t* codes, const __nv_bfloat16* scales, const uint8_t* zeros,
                       int64_t N, int64_t K, int g, int bits, __nv_bfloat16* out, cudaStream_t st) {
    const int64_t chunks = N * K / 8;
    if (chunks == 0) return;
    k_dequantize<<<(unsigned)((chunks + 255) / 256), 256, 0, st>>>(codes, scales, zeros, N, K, g, bits, out);
}

// slot image -> slot image (both in the pair-interleaved packing)
void launch_quantize_slot(const uint8_t* src_slot, const SlotLayout& src, uint8_t* dst_slot,
                          const SlotLayout& dst, int H, int I, int g, cudaStream_t st) {
    const int64_t rows[3] = {I, I, H}, cols[3] = {H, H, I};
    for (int m = 0; m < 3; ++m) {
        const uint8_t* s_codes = src_slot + m * src.codes_stride;
        const uint8_t* s_sc = src.bits == 16 ? nullptr : src_slot + src.scales_off + m * src.scales_stride;
        const uint8_t* s_z = src.bits == 16 ? nullptr : src_slot + src.zeros_off + m * src.zeros_stride;
        quantize_impl(s_codes, src.bits, s_sc, s_z, rows[m], cols[m], g, dst.bits, dst_slot + m * dst.codes_stride,
                      reinterpret_cast<__nv_bfloat16*>(dst_slot + dst.scales_off + m * dst.scales_stride),
                      dst_slot + dst.zeros_off + m * dst.zeros_stride, 1, 1, st);
    }
}
