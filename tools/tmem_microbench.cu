// tmem_microbench.cu -- TMEM read throughput of tcgen05.ld.32x32b.x32 per SM sub-partition, as a function of the
// number of warps per sub-partition and of how many loads are in flight before tcgen05.wait::ld.
// Design input for the softmax pass structure of attn_fwd.cu (two passes over S read it twice).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_12056_b200/csrc -I tools tools/tmem_microbench.cu -o tools/tmem_mb.bin
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx_cta1.cuh"

using namespace spa;
constexpr int ITER = 512;

template <int INFLIGHT>
__global__ void tmem_ld_kernel(int warps_per_smsp, unsigned long long *cycles, uint32_t *sink) {
    __shared__ uint32_t base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        ptx::tmem_alloc(&base, 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t t = base + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long c0 = clock64();
    if (warp < 4 * warps_per_smsp) {
        for (int it = 0; it < ITER; ++it) {
#pragma unroll
            for (int k = 0; k < 4; k += INFLIGHT) {
                uint32_t r[INFLIGHT][32];
#pragma unroll
                for (int u = 0; u < INFLIGHT; ++u) ptx::tmem_ld32(t + 32 * ((k + u + warp) & 15), r[u]);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int u = 0; u < INFLIGHT; ++u)
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc ^= r[u][i];
            }
        }
    }
    __syncthreads();
    const unsigned long long c1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(base, 512);
    }
}

template <int INFLIGHT>
void run(int wps) {
    unsigned long long *c;
    uint32_t *s;
    cudaMalloc(&c, 148 * 8);
    cudaMalloc(&s, 148 * 512 * 4);
    for (int rep = 0; rep < 2; ++rep) tmem_ld_kernel<INFLIGHT><<<148, 512>>>(wps, c, s);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148; ++i) mean += h[i] / 148.0;
    // bytes per SMSP: warps_per_smsp warps x ITER x 4 loads x 32 lanes x 32 cols x 4 B
    const double bytes = (double)wps * ITER * 4 * 32 * 32 * 4;
    printf("{\"inflight\": %d, \"warps_per_smsp\": %d, \"cycles\": %.0f, \"bytes_per_cycle_per_smsp\": %.1f, "
           "\"cycles_per_x32_load\": %.1f}\n",
           INFLIGHT, wps, mean, bytes / mean, mean / (wps * ITER * 4.0));
    cudaFree(c);
    cudaFree(s);
}

int main() {
    for (int w = 1; w <= 4; ++w) run<1>(w);
    for (int w = 1; w <= 4; ++w) run<2>(w);
    for (int w = 1; w <= 4; ++w) run<4>(w);
    cudaError_t e = cudaGetLastError();
    printf("{\"cuda\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
