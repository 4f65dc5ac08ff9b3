// tma_probe.cu -- microbenchmark: HBM streaming rate of TMA tile loads for two weight layouts.
//   (a) row-major [rows][2048] bf16, K-major 128-row x 64-col boxes (128 B per row, 4 KB apart)
//   (b) tiled: every 128 x 64 tile stored contiguously (16 KB), same boxes
//   (c) row-major, 16-row boxes x 8 (the gate/up interleave of k_gemm)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_15015_b200/csrc
//        scripts/tma_probe.cu -o tma_probe -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "dx_sm100.cuh"
using namespace sm100;

constexpr int STAGES = 8, TILE = 16384;

__global__ void __launch_bounds__(128, 1) k_stream(const __grid_constant__ CUtensorMap map, int mode, int ntiles_total,
                                                   int nk, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(buf + STAGES * TILE);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    // tiles assigned round-robin: tile id t -> (m-block, k-block) = (t / nk, t % nk)
    int issued = 0, done = 0;
    unsigned long long acc = 0;
    const int my = (ntiles_total - blockIdx.x + gridDim.x - 1) / gridDim.x;
    auto issue = [&](int i) {
        const int t = blockIdx.x + i * gridDim.x;
        const int st = i % STAGES;
        mbar_arrive_expect_tx(&full[st], TILE);
        const int mb = t / nk, kb = t % nk;
        if (mode == 0) tma_load_3d(buf + st * TILE, &map, &full[st], kb * 64, mb * 128, 0);
        else if (mode == 1) tma_load_3d(buf + st * TILE, &map, &full[st], 0, 0, t);
        else
            for (int j = 0; j < 8; ++j) tma_load_3d(buf + st * TILE + j * 2048, &map, &full[st], kb * 64, mb * 128 + 16 * j, 0);
    };
    for (; issued < STAGES && issued < my; ++issued) issue(issued);
    for (; done < my; ++done) {
        const int st = done % STAGES;
        mbar_wait(&full[st], (done / STAGES) & 1);
        acc += buf[st * TILE + (done & 1023)];
        if (issued < my) issue(issued++);
    }
    if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
    const size_t rows = 128ull * 1024, K = 2048;            // 512 MB of bf16 weights
    const size_t bytes = rows * K * 2;
    void* d;
    cudaMalloc(&d, bytes);
    cudaMemset(d, 1, bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    void* fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    const int nk = K / 64, ntiles = (rows / 128) * nk;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * TILE + 2048);
    for (int mode = 0; mode < 3; ++mode) {
        CUtensorMap m;
        uint32_t es[3] = {1, 1, 1};
        if (mode == 1) {
            uint64_t dims[3] = {64, 128, (uint64_t)ntiles}, str[2] = {128, TILE};
            uint32_t box[3] = {64, 128, 1};
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            uint64_t dims[3] = {K, rows, 1}, str[2] = {K * 2, bytes};
            uint32_t box[3] = {64, (uint32_t)(mode == 0 ? 128 : 16), 1};
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            k_stream<<<148, 128, STAGES * TILE + 2048>>>(m, mode, ntiles, nk, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("mode %d (%s): %.1f GB/s\n", mode, mode == 0 ? "row-major 128-row box" : mode == 1 ? "tiled 16 KB" : "row-major 8x16-row boxes",
                            bytes / ms / 1e6);
        }
        printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    }
    return 0;
}
