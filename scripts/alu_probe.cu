// ALU throughput probe (sm_100a): warp-instructions per cycle per SMSP for the dequant's instruction mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_probe alu_probe.cu && ./alu_probe
#include <cstdio>
#include <cuda_bf16.h>
#include <cstdint>

template <int OP>
__global__ void probe(uint32_t* out, int iters, uint32_t seed) {
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = seed * (threadIdx.x + 1) + i * 0x01010101u;
    uint32_t zz = 0x43084308u, ss = 0x3c003c00u;
    asm volatile("" : "+r"(zz), "+r"(ss));
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (OP == 0) asm volatile("fma.rn.bf16x2 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(ss), "r"(zz));
            if (OP == 1) asm volatile("mul.rn.bf16x2 %0, %0, %1;" : "+r"(r[i]) : "r"(ss));
            if (OP == 2) { float f = __uint_as_float(r[i]); asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f) : "f"(1.0001f), "f"(0.5f)); r[i] = __float_as_uint(f); }
            if (OP == 3) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(r[i]) : "r"(0x000F000Fu), "r"(0x43004300u));
            if (OP == 4) asm volatile("sub.rn.bf16x2 %0, %0, %1;" : "+r"(r[i]) : "r"(zz));
            if (OP == 5) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(ss), "r"(zz));
            if (OP == 6) { asm volatile("{\n.reg .b32 t;\nsub.rn.bf16x2 t, %0, %1;\nmul.rn.bf16x2 %0, t, %2;\n}" : "+r"(r[i]) : "r"(zz), "r"(ss)); }
        }
    }
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc ^= r[i];
    if (acc == 0x12345u) out[1] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (uint32_t)(t1 - t0);
}

template <int OP>
void run(const char* name, int warps) {
    uint32_t* d;
    cudaMalloc(&d, 64);
    const int iters = 4096;
    probe<OP><<<1, 32 * warps>>>(d, iters, 7);
    probe<OP><<<1, 32 * warps>>>(d, iters, 7);
    uint32_t cyc;
    cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
    const double instr_per_smsp = (double)iters * 16 * warps / 4;   // warp-instructions issued per SMSP
    const int n_ops = OP == 6 ? 2 : 1;
    printf("%-28s warps %2d: %.3f warp-instr/cycle/SMSP\n", name, warps, instr_per_smsp * n_ops / cyc);
    cudaFree(d);
}

int main() {
    for (int w : {4, 16}) {
        run<0>("fma.rn.bf16x2", w);
        run<1>("mul.rn.bf16x2", w);
        run<4>("sub.rn.bf16x2", w);
        run<5>("fma.rn.f16x2", w);
        run<2>("fma.rn.f32", w);
        run<3>("lop3", w);
        run<6>("sub+mul bf16x2", w);
    }
    return 0;
}
