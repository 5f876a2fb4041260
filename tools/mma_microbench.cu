// mma_microbench.cu -- raw tcgen05.mma issue rates on this B200 (design input for attn_fwd.cu).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_12056_b200/csrc -I tools tools/mma_microbench.cu -o /tmp/mma_mb
// One elected thread per CTA issues ITER back-to-back MMAs (random bf16 operands), commit, wait.
// Prints cycles per MMA instruction and the implied bf16 FLOP/clk/SM, for 1 CTA and for 148 CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx_cta1.cuh"

using namespace spa;

constexpr int ITER = 4096;

template <int MODE>
__global__ void __launch_bounds__(128, 1) mb_kernel(unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    // fill 128 KB with pseudo-random bf16 in [-1, 1)
    uint32_t *w = reinterpret_cast<uint32_t *>(smem);
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) {
        uint32_t x = i * 2654435761u + blockIdx.x * 97u;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        uint32_t lo = 0x3c00u | (x & 0x7f) | ((x >> 7 & 1) << 15);
        uint32_t hi = 0x3c00u | (x >> 8 & 0x7f) | ((x >> 15 & 1) << 15);
        w[i] = lo | (hi << 16);
    }
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (threadIdx.x < 32) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = tbase;
    const uint32_t sa = ptx::smem_u32(smem);
    if (threadIdx.x == 0) {
        uint64_t t0 = clock64();
        for (int i = 0; i < ITER; ++i) {
            const uint32_t kk = i & 3;
            if (MODE == 0) {        // SS M128 N128 K16
                ptx::mma_ss(tm, ptx::smem_desc(sa + kk * 32, 16, 1024, 2), ptx::smem_desc(sa + 32768 + kk * 32, 16, 1024, 2),
                            ptx::idesc_bf16(128, 128, 0, 0), 1);
            } else if (MODE == 1) { // SS M128 N256 K16
                ptx::mma_ss(tm, ptx::smem_desc(sa + kk * 32, 16, 1024, 2), ptx::smem_desc(sa + 32768 + kk * 32, 16, 1024, 2),
                            ptx::idesc_bf16(128, 256, 0, 0), 1);
            } else if (MODE == 2) { // TS M128 N128 (B MN-major, two 64-col atoms 16 KB apart)
                ptx::mma_ts(tm + 256, tm + kk * 8, ptx::smem_desc(sa + kk * 2048, 16384, 1024, 2),
                            ptx::idesc_bf16(128, 128, 0, 1), 1);
            } else if (MODE == 3) { // TS M128 N64
                ptx::mma_ts(tm + 256, tm + kk * 8, ptx::smem_desc(sa + kk * 2048, 16, 1024, 2),
                            ptx::idesc_bf16(128, 64, 0, 1), 1);
            } else if (MODE == 4) { // SS M128 N64
                ptx::mma_ss(tm, ptx::smem_desc(sa + kk * 32, 16, 1024, 2), ptx::smem_desc(sa + 32768 + kk * 32, 16, 1024, 2),
                            ptx::idesc_bf16(128, 64, 0, 0), 1);
            } else if (MODE == 5) { // SS M128 N128, B MN-major (V-like)
                ptx::mma_ss(tm, ptx::smem_desc(sa + kk * 32, 16, 1024, 2), ptx::smem_desc(sa + 32768 + kk * 2048, 16384, 1024, 2),
                            ptx::idesc_bf16(128, 128, 0, 1), 1);
            }
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        uint64_t t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    if (threadIdx.x < 32) ptx::tmem_dealloc(tm, 512);
}

template <int MODE>
void run(const char *name, int N, int flops_per) {
    unsigned long long *d, h[148];
    cudaMalloc(&d, sizeof(h));
    cudaFuncSetAttribute(mb_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    for (int nct : {1, 148}) {
        mb_kernel<MODE><<<nct, 128, 140 * 1024>>>(d);
        mb_kernel<MODE><<<nct, 128, 140 * 1024>>>(d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
        cudaMemcpy(h, d, nct * 8, cudaMemcpyDeviceToHost);
        double s = 0; for (int i = 0; i < nct; ++i) s += h[i]; s /= nct;
        printf("%-28s ctas=%3d  cycles/mma=%7.2f  flop/clk/SM=%7.0f\n", name, nct, s / ITER, flops_per / (s / ITER));
    }
    cudaFree(d);
}

int main() {
    run<0>("SS M128 N128 K16", 0, 2 * 128 * 128 * 16);
    run<1>("SS M128 N256 K16", 0, 2 * 128 * 256 * 16);
    run<2>("TS M128 N128 K16 (Bmn)", 0, 2 * 128 * 128 * 16);
    run<3>("TS M128 N64 K16 (Bmn)", 0, 2 * 128 * 64 * 16);
    run<4>("SS M128 N64 K16", 0, 2 * 128 * 64 * 16);
    run<5>("SS M128 N128 K16 (Bmn)", 0, 2 * 128 * 128 * 16);
    return 0;
}
