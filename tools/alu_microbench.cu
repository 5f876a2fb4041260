// alu_microbench.cu -- per-SMSP throughput of the softmax instruction mix (MUFU.EX2, FFMA, FFMA2,
// F2FP bf16x2 pack, FMNMX) with one warp per SMSP, 16 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/alu_microbench.cu -o tools/alu_mb.bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITER = 2048;
constexpr int NCH = 16;

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(float *out, unsigned long long *cyc, float seed) {
    float a[NCH];
    uint32_t u[NCH];
#pragma unroll
    for (int i = 0; i < NCH; ++i) { a[i] = seed * (i + 1) * 1e-3f - 1.0f; u[i] = i; }
    const float c1 = 1.0001f, c2 = -0.5f;
    __syncthreads();
    uint64_t t0 = clock64();
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            if (MODE == 1) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(c1), "f"(c2));
            if (MODE == 2) {  // packed fma on two lanes of a 64-bit pair
                if (i & 1) continue;
                asm volatile("{.reg .b64 x, y, z; mov.b64 x, {%0, %1}; mov.b64 y, {%2, %2}; mov.b64 z, {%3, %3};"
                             "fma.rn.f32x2 x, x, y, z; mov.b64 {%0, %1}, x;}"
                             : "+f"(a[i]), "+f"(a[i + 1]) : "f"(c1), "f"(c2));
            }
            if (MODE == 3) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(u[i]) : "f"(a[i]), "f"(__uint_as_float(u[i])));
            if (MODE == 4) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(c1));
            if (MODE == 5) {  // mixed: 1 ex2 + 1 ffma + 1 fadd + 0.5 pack per element (softmax-like)
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(c1), "f"(c2));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(c2));
                if (i & 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(u[i]) : "f"(a[i]), "f"(a[i - 1]));
            }
            if (MODE == 6) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i]));
            if (MODE == 7) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(c2));
        }
    }
    uint64_t t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < NCH; ++i) s += a[i] + __uint_as_float(u[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char *name, double ops_per_thread_iter) {
    float *o; unsigned long long *c, h[148];
    cudaMalloc(&o, 148 * 128 * 4); cudaMalloc(&c, sizeof(h));
    for (int rep = 0; rep < 2; ++rep) k<MODE><<<148, 128>>>(o, c, 1.0f);
    cudaDeviceSynchronize();
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148; ++i) s += h[i]; s /= 148;
    double instr = ITER * ops_per_thread_iter;   // warp-instructions per warp
    printf("%-34s cycles/warp-instr/SMSP = %6.2f   lanes/clk/SM = %6.1f\n", name, s / instr, 4 * 32 / (s / instr));
    cudaFree(o); cudaFree(c);
}

int main() {
    run<0>("MUFU ex2.approx.ftz.f32", NCH);
    run<6>("MUFU ex2.approx.f16x2", NCH);
    run<1>("FFMA (3 reg)", NCH);
    run<2>("FFMA2 fma.rn.f32x2 (per instr)", NCH / 2);
    run<3>("F2FP cvt.rn.bf16x2.f32", NCH);
    run<4>("FMNMX", NCH);
    run<7>("FADD", NCH);
    run<5>("mix (per element: ffma+ex2+fadd+.5cvt)", NCH * 3.5);
    return 0;
}
