// q_probe2.cu -- int4 decode pipeline microbenchmark, round-robin transform groups: the NTW dequant warps form
// RR groups and group g dequantises whole stages s = g (mod RR), so one group's waits (stage landing, TMEM buffer
// free, store completion) overlap the other groups' arithmetic.  RR = 1 is the round-1 split (every group one
// chunk of every stage).  Flat fp32 accumulator per item (N = 32 tokens), exact dequant bf16_rn((q - z) s).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_15015_b200/csrc \
//        scripts/q_probe2.cu -o scripts/q_probe2 -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "dx_sm100.cuh"
using namespace sm100;

#ifndef NTOK_V
#define NTOK_V 32
#endif
constexpr int KTOT = 2048, NTOK = NTOK_V, G = 16;
constexpr int CODE_BYTES = 16384, B_BYTES = NTOK * 256 * 2;
constexpr int TAB = 128 * G * 3;

__device__ __forceinline__ uint32_t and_or(uint32_t x, uint32_t m, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(x), "r"(m), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t deq2(uint32_t q128, uint32_t zz, uint32_t ss) {
    uint32_t d;
    asm("{\n.reg .b32 t;\nsub.rn.bf16x2 t, %1, %2;\nmul.rn.bf16x2 %0, t, %3;\n}" : "=r"(d) : "r"(q128), "r"(zz), "r"(ss));
    return d;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    const uint32_t a = smem_u32(b);
    for (uint32_t n = 0; !mbar_try_wait(a, ph); ++n)
        if (n > (1u << 26)) __trap();
}

template <int CS, int BS, int NTW, int RR, int NA, int MATH>
__global__ void __launch_bounds__(32 * (NTW + 6), 1)
k_probe(const __grid_constant__ CUtensorMap cmap, const __grid_constant__ CUtensorMap bmap, const uint8_t* tabs_g,
        int n_it, float* out) {
    constexpr int WPG = NTW / RR;                 // warps per group
    constexpr int WPQ = WPG / 4;                  // warps per TMEM lane quarter per group
    constexpr int CPW = 4 / WPQ;                  // chunks per warp per stage
    constexpr int W_EPI = 2 + NTW;
    static_assert(WPQ >= 1 && 4 % WPQ == 0, "shape");
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sC = sm;
    uint8_t* sB = sC + CS * CODE_BYTES;
    uint8_t* sT = sB + BS * B_BYTES;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sT + 2 * TAB);
    uint64_t *cfull = bar, *cempty = cfull + CS, *bfull = cempty + CS, *bempty = bfull + BS, *aready = bempty + BS,
             *aempty = aready + NA, *tfull = aempty + NA, *tempty = tfull + 2, *tabfull = tempty + 2, *tabempty = tabfull + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tabempty + 2);
    const int warp = __shfl_sync(~0u, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < CS; ++s) { mbar_init(&cfull[s], 1); mbar_init(&cempty[s], WPG); }
        for (int s = 0; s < BS; ++s) { mbar_init(&bfull[s], 1); mbar_init(&bempty[s], 1); }
        for (int s = 0; s < NA; ++s) { mbar_init(&aready[s], WPG); mbar_init(&aempty[s], 1); }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 4);
            mbar_init(&tabfull[s], 1); mbar_init(&tabempty[s], NTW);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t tmem_a = tmem + 64;
    constexpr int nst = KTOT / 256;
    if (warp == 0) {
        if (elect_one()) {
            int cs = 0, bs = 0;
            uint32_t cph = 0, bph = 0;
            for (int i = 0; i < n_it; ++i) {
                const int item = blockIdx.x * n_it + i;
                const int tb = i & 1;
                wait(&tabempty[tb], ((i >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&tabfull[tb], TAB);
                bulk_load(sT + tb * TAB, tabs_g + (size_t)item * TAB, TAB, &tabfull[tb]);
                for (int kb = 0; kb < nst; ++kb) {
                    wait(&cempty[cs], cph ^ 1);
                    mbar_arrive_expect_tx(&cfull[cs], CODE_BYTES);
                    tma_load_2d(sC + cs * CODE_BYTES, &cmap, &cfull[cs], kb * 128, item * 128);
                    wait(&bempty[bs], bph ^ 1);
                    mbar_arrive_expect_tx(&bfull[bs], B_BYTES);
                    tma_load_3d(sB + bs * B_BYTES, &bmap, &bfull[bs], 0, 0, kb * 4);
                    if (++cs == CS) { cs = 0; cph ^= 1; }
                    if (++bs == BS) { bs = 0; bph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        int bs = 0, ab = 0;
        uint32_t bph = 0, aph = 0;
        const uint32_t idesc = idesc_bf16(128, NTOK);
        for (int i = 0; i < n_it; ++i) {
            const int buf = i & 1;
            wait(&tempty[buf], ((i >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + buf * 32;
            for (int kb = 0; kb < nst; ++kb) {
                wait(&bfull[bs], bph);
                wait(&aready[ab], aph);
                tc_fence_after();
                const uint64_t db = umma_desc_sw128(smem_u32(sB + bs * B_BYTES));
                const uint32_t bstep = (NTOK * 128) >> 4;
                const uint32_t at = tmem_a + ab * 128;
                if (elect_one()) {
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        mma_bf16_ts(d, at + 8 * q, db + (q >> 2) * bstep + 2 * (q & 3), idesc, (kb | q) != 0);
                    mma_commit(&aempty[ab]);
                    mma_commit(&bempty[bs]);
                }
                __syncwarp();
                if (++bs == BS) { bs = 0; bph ^= 1; }
                if (++ab == NA) { ab = 0; aph ^= 1; }
            }
            if (elect_one()) mma_commit(&tfull[buf]);
            __syncwarp();
        }
    } else if (warp < W_EPI) {
        const int gid = (warp - 2) >> 2, qa = warp & 3, r = 32 * qa + lane;
        const int group = gid % RR, sub = gid / RR;
        const uint32_t rsw = r & 7;
        const uint32_t lane_base = tmem_a + ((uint32_t)(32 * qa) << 16);
        uint32_t magic = 0x43004300u;
        asm volatile("" : "+r"(magic));
        const int n_st = n_it * nst;
        for (int s = group; s < n_st; s += RR) {
            const int i = s / nst, kb = s % nst;
            const int cs = s % CS, ab = s % NA;
            const uint32_t cph = (s / CS) & 1, aph = (s / NA) & 1;
            const int tb = i & 1;
            if (s - RR < i * nst) wait(&tabfull[tb], (i >> 1) & 1);      // first stage of item i for this warp
            const uint32_t tsc = smem_u32(sT + tb * TAB) + r * G * 2, tze = smem_u32(sT + tb * TAB + 128 * G * 2) + r * G;
            wait(&cfull[cs], cph);
            const uint32_t row = smem_u32(sC + cs * CODE_BYTES) + r * 128;
            uint32_t src[CPW][8];
#pragma unroll
            for (int h = 0; h < CPW; ++h) {
                const uint32_t c = 2 * (sub * CPW + h);
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(src[h][0]), "=r"(src[h][1]), "=r"(src[h][2]), "=r"(src[h][3])
                             : "r"(row + ((c ^ rsw) << 4)));
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(src[h][4]), "=r"(src[h][5]), "=r"(src[h][6]), "=r"(src[h][7])
                             : "r"(row + (((c + 1) ^ rsw) << 4)));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&cempty[cs]);
            wait(&aempty[ab], aph ^ 1);
            tc_fence_after();
#pragma unroll
            for (int h = 0; h < CPW; ++h) {
                const int j = sub * CPW + h;
                const int gi = (kb * 256 + j * 64) >> 7;
                uint16_t sv, zv;
                asm volatile("ld.shared.u16 %0, [%1];" : "=h"(sv) : "r"(tsc + 2 * gi));
                asm volatile("ld.shared.u8 %0, [%1];" : "=h"(zv) : "r"(tze + gi));
                const uint32_t ss = (uint32_t)sv * 0x10001u, zz = (0x4300u + zv) * 0x10001u;
                uint32_t wv[32];
                if (MATH == 1) {
#pragma unroll
                    for (int b = 0; b < 32; ++b)
                        wv[b] = deq2(and_or(src[h][b >> 2] >> (4 * (b & 3)), 0x000F000Fu, magic), zz, ss);
                } else {
#pragma unroll
                    for (int b = 0; b < 32; ++b) wv[b] = src[h][b >> 2] ^ zz ^ ss;
                }
                tmem_st32(lane_base + ab * 128 + 32 * j, wv);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&aready[ab]);
                if ((s + RR) / nst != i) mbar_arrive(&tabempty[tb]);     // last stage of item i for this warp
            }
        }
    } else {
        const int q = warp & 3;
        for (int i = 0; i < n_it; ++i) {
            const int buf = i & 1;
            wait(&tfull[buf], (i >> 1) & 1);
            tc_fence_after();
            uint32_t v[32];
            tmem_ld32(tmem + buf * 32 + ((uint32_t)(32 * q) << 16), v);
            tmem_ld_wait();
            float s = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) s += __uint_as_float(v[j]);
            out[(size_t)(blockIdx.x * n_it + i) * 128 + 32 * q + lane] = s;
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int CS, int BS, int NTW, int RR, int NA, int MATH>
void run(const CUtensorMap& cm, const CUtensorMap& bm, const uint8_t* tabs, int ipc, float* out, int ctas, double bytes) {
    constexpr int SMEM = 1024 + CS * CODE_BYTES + BS * B_BYTES + 2 * TAB + 1024;
    auto k = k_probe<CS, BS, NTW, RR, NA, MATH>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess) {
        printf("smem %d too big\n", SMEM);
        cudaGetLastError();
        return;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 2; ++w) k<<<ctas, 32 * (NTW + 6), SMEM>>>(cm, bm, tabs, ipc, out);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int w = 0; w < reps; ++w) k<<<ctas, 32 * (NTW + 6), SMEM>>>(cm, bm, tabs, ipc, out);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("CS=%2d BS=%d NTW=%2d RR=%d NA=%d math=%d : %7.1f us  %6.0f GB/s  (%s)\n", CS, BS, NTW, RR, NA, MATH,
           ms * 1e3 / reps, bytes * reps / (ms * 1e6), cudaGetErrorString(err));
    if (err != cudaSuccess) exit(1);
}

int main(int argc, char** argv) {
    const int ctas = 148, ipc = argc > 1 ? atoi(argv[1]) : 8;
    const int n_items = ctas * ipc;
    const size_t code_bytes = (size_t)n_items * 128 * (KTOT / 2);
    uint8_t *codes, *tabs, *x;
    float* out;
    cudaMalloc(&codes, code_bytes);
    cudaMemset(codes, 0x5a, code_bytes);
    cudaMalloc(&tabs, (size_t)n_items * TAB);
    cudaMemset(tabs, 0x3c, (size_t)n_items * TAB);
    cudaMalloc(&x, (size_t)NTOK * KTOT * 2);
    cudaMemset(x, 0x3c, (size_t)NTOK * KTOT * 2);
    cudaMalloc(&out, (size_t)n_items * 128 * 4);
    void* fn;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap cm, bm;
    uint32_t es[3] = {1, 1, 1};
    {
        uint64_t dims[2] = {KTOT / 2, (uint64_t)n_items * 128}, str[1] = {KTOT / 2};
        uint32_t box[2] = {128, 128};
        enc(&cm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, codes, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    {
        uint64_t dims[3] = {64, NTOK, KTOT / 64}, str[2] = {KTOT * 2, 128};
        uint32_t box[3] = {64, NTOK, 4};
        enc(&bm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    const double bytes = (double)code_bytes + (double)n_items * TAB;
    printf("items %d (%d per CTA), %.1f MB of codes + tables per launch\n", n_items, ipc, bytes / 1e6);
    run<8, 4, 16, 1, 3, 1>(cm, bm, tabs, ipc, out, ctas, bytes);
    run<8, 4, 16, 2, 3, 1>(cm, bm, tabs, ipc, out, ctas, bytes);
    run<6, 4, 16, 2, 3, 1>(cm, bm, tabs, ipc, out, ctas, bytes);
    return 0;
}
