// tma_microbench.cu -- L2 -> SMEM delivery rate of TMA tile loads per SM, the way attn_fwd.cu streams K/V:
// 128-row x 128-col bf16 tiles (32 KB, four 64x64 SW128 boxes) from a strided [rows][heads*D] array through
// an NS-slot ring; a consumer thread frees each slot as soon as it lands (no compute).
//   mode 0: no cluster, each CTA loads whole tiles
//   mode 1: clusters of 2, each CTA loads half of every tile and multicasts it (attn_fwd's scheme)
// Reports bytes landed in each SM's shared memory per SM clock.  Design input for the attention kernel's
// structure (how many query rows must share one K/V tile).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_12056_b200/csrc -I tools tools/tma_microbench.cu -o tools/tma_mb.bin -lcuda
#include <cuda.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx_cta1.cuh"

using namespace spa;
constexpr int NS = 6;
constexpr int TILE = 128 * 128 * 2;
constexpr int ROWS = 32768;
constexpr int TILES = 256;  // per CTA

template <int CLM>
__global__ void __launch_bounds__(64, 1) tma_kernel(const __grid_constant__ CUtensorMap tm, unsigned long long *cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[NS], empty[NS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], CLM);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (CLM > 1) ptx::cluster_sync();
    const uint32_t crank = CLM > 1 ? ptx::cluster_ctarank() : 0;
    const int start = (blockIdx.x / CLM) * 7 % (ROWS / 128);
    const unsigned long long c0 = clock64();
    if (warp == 0 && lane == 0) {
        const uint64_t pol = ptx::policy_evict_last();
        for (int i = 0; i < TILES; ++i) {
            const int slot = i % NS;
            ptx::mbar_wait(&empty[slot], ((i / NS) & 1) ^ 1);
            ptx::mbar_arrive_expect_tx(&full[slot], TILE);
            const int row0 = ((start + i) % (ROWS / 128)) * 128;
            uint8_t *dst = sm + slot * TILE;
            for (int c = 0; c < 2; ++c) {        // two 64-column chunks
                if (CLM == 1) {
                    for (int h = 0; h < 2; ++h)
                        ptx::tma_load_4d(&tm, &full[slot], dst + c * 16384 + h * 8192, c * 64, 0, row0 + h * 64, 0, pol);
                } else {
                    ptx::tma_load_4d_mc(&tm, &full[slot], dst + c * 16384 + crank * 8192, c * 64, 0,
                                        row0 + (int)crank * 64, 0, 0x3, pol);
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int i = 0; i < TILES; ++i) {
            const int slot = i % NS;
            ptx::mbar_wait(&full[slot], (i / NS) & 1);
            if (CLM == 1) ptx::mbar_arrive(&empty[slot]);
            else {
                // arrive on the empty barrier of every CTA of the pair (both must be done before a reload)
                for (uint32_t r = 0; r < 2; ++r) {
                    uint32_t remote;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(ptx::smem_u32(&empty[slot])), "r"(r));
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
                }
            }
        }
    }
    __syncthreads();
    const unsigned long long c1 = clock64();
    if (CLM > 1) ptx::cluster_sync();
    if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int CLM>
void run(void *buf, int heads, int D, int grid) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(p);
    CUtensorMap tm;
    cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)heads, (cuuint64_t)ROWS, 1};
    cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)heads * D * 2, (cuuint64_t)ROWS * heads * D * 2};
    cuuint32_t box[4] = {64, 1, 64, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("{\"error\": \"encode %d\"}\n", (int)r); return; }
    unsigned long long *cyc;
    cudaMalloc(&cyc, grid * 8);
    const int smem = NS * TILE + 1024;
    cudaFuncSetAttribute(tma_kernel<CLM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CLM;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, tma_kernel<CLM>, tm, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    unsigned long long h[1024];
    cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < grid; ++i) mean += (double)h[i] / grid;
    const double bytes_sm = (double)TILES * TILE;   // landed in each SM's smem
    printf("{\"cluster\": %d, \"grid\": %d, \"row_bytes\": %d, \"cycles\": %.0f, \"bytes_per_cycle_per_sm\": %.1f, "
           "\"ms\": %.3f, \"chip_smem_fill_GBps\": %.0f, \"l2_read_GBps\": %.0f}\n",
           CLM, grid, heads * D * 2, mean, bytes_sm / mean, best, bytes_sm * grid / best / 1e6,
           bytes_sm * grid / CLM / best / 1e6);
    cudaFree(cyc);
}

int main() {
    void *buf;
    const int heads = 3, D = 128;
    cudaMalloc(&buf, (size_t)ROWS * heads * D * 2);
    cudaMemset(buf, 0, (size_t)ROWS * heads * D * 2);
    for (int g : {148, 296}) {
        run<1>(buf, heads, D, g);
        run<2>(buf, heads, D, g);
    }
    printf("{\"cuda\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
