// mma_probe.cu -- microbenchmark: cost of back-to-back tcgen05.mma (kind::f16, M = 128, K = 16) issued by
// one thread, by form (SS: A and B in smem / TS: A in TMEM), N, accumulator chaining and issue style.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_15015_b200/csrc
//        scripts/mma_probe.cu -o scripts/mma_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "dx_sm100.cuh"
using namespace sm100;

// mode bit0: TS (A in TMEM) else SS; bit1: 4 independent accumulators; bit2: whole warp runs the loop,
// one elected lane issues
__global__ void __launch_bounds__(128, 1) k_probe(int mode, int n_mma, int N, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(buf)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    fence_proxy_async_smem();
    if (threadIdx.x < 32) tmem_alloc<512>(slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t idesc = idesc_bf16(128, N);
    const uint32_t sA = smem_u32(buf), sB = sA + 16384;
    const uint64_t da = umma_desc_sw128(sA), db = umma_desc_sw128(sB);
    const bool ts = mode & 1, multi = mode & 2, warpwide = mode & 4;
    if (mode & 16) {
        // uniform values computed by the whole warp, the whole loop inside one elected lane
        const int wi = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        if (wi == 0) {
            uint32_t p;
            asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}" : "=r"(p));
            if (p) {
                const unsigned long long t0 = clock64();
#pragma unroll 4
                for (int i = 0; i < n_mma; ++i) {
                    const uint32_t d = tm + ((mode & 2) ? (i & 3) * N : 0);
                    const int s = i & 3;
                    if (ts) mma_bf16_ts(d, tm + 256 + 8 * s, db + 2 * s, idesc, 1);
                    else mma_bf16(d, da + 2 * s, db + 2 * s, idesc, 1);
                }
                const unsigned long long t1 = clock64();
                mma_commit(bar);
                mbar_wait(bar, 0);
                const unsigned long long t2 = clock64();
                out[2 * blockIdx.x] = t1 - t0;
                out[2 * blockIdx.x + 1] = t2 - t0;
            }
        }
    } else if (mode & 8) {
        // warp index and TMEM base made provably warp-uniform (shfl), whole warp runs the loop, one elected
        // lane issues: the compiler keeps descriptors in uniform registers
        const int wi = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        if (wi == 0) {
            const unsigned long long t0 = clock64();
#pragma unroll 4
            for (int i = 0; i < n_mma; ++i) {
                const uint32_t d = tm + ((mode & 2) ? (i & 3) * N : 0);
                const int s = i & 3;
                uint32_t p;
                asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}" : "=r"(p));
                if (p) {
                    if (ts) mma_bf16_ts(d, tm + 256 + 8 * s, db + 2 * s, idesc, 1);
                    else mma_bf16(d, da + 2 * s, db + 2 * s, idesc, 1);
                }
            }
            const unsigned long long t1 = clock64();
            if (threadIdx.x == 0) {
                mma_commit(bar);
                mbar_wait(bar, 0);
                const unsigned long long t2 = clock64();
                out[2 * blockIdx.x] = t1 - t0;
                out[2 * blockIdx.x + 1] = t2 - t0;
            }
        }
    } else if (threadIdx.x < 32 && (warpwide || threadIdx.x == 0)) {
        const unsigned long long t0 = clock64();
        for (int i = 0; i < n_mma; ++i) {
            const uint32_t d = tmem + (multi ? (i & 3) * N : 0);
            const int s = i & 3;
            bool leader = true;
            if (warpwide) {
                uint32_t p;
                asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}" : "=r"(p));
                leader = p;
            }
            if (leader) {
                if (ts) mma_bf16_ts(d, tmem + 256 + 8 * s, db + 2 * s, idesc, 1);
                else mma_bf16(d, da + 2 * s, db + 2 * s, idesc, 1);
            }
        }
        const unsigned long long t1 = clock64();
        if (threadIdx.x == 0) {
            mma_commit(bar);
            mbar_wait(bar, 0);
            const unsigned long long t2 = clock64();
            out[2 * blockIdx.x] = t1 - t0;
            out[2 * blockIdx.x + 1] = t2 - t0;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 2 * 148 * sizeof(unsigned long long));
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    const int n = 4096;
    printf("mode: bit0 TS, bit1 4 accumulators, bit2 warp-wide loop + elect;  cycles per MMA (issue / complete)\n");
    for (int mode : {8, 9, 16, 17, 18, 19})
        for (int N : {16, 64, 128}) {
            if ((mode & 2) && N > 64) continue;
            k_probe<<<148, 128, 40000>>>(mode, n, N, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            unsigned long long h[2 * 148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double iss = 0, tot = 0;
            for (int b = 0; b < 148; ++b) { iss += h[2 * b]; tot += h[2 * b + 1]; }
            printf("mode %d (%s%s%s) N=%3d: %7.1f / %7.1f\n", mode, mode & 1 ? "TS" : "SS", mode & 2 ? " 4acc" : "",
                   mode & 4 ? " warp" : mode & 8 ? " uniform" : mode & 16 ? " uniform-in-elect" : "", N, iss / 148 / n, tot / 148 / n);
        }
    return 0;
}
