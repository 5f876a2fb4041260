// mma_interference.cu -- does issuing tcgen05.mma from a warp slow the softmax warps that share its SM sub-partition?
// The attention kernel's per-warp trace shows the leader CTA's lane-quarter-3 softmax warps (the SMSP of the MMA-issuing
// warp) ~15 % slower than the other quarters.  Layout as in attn_fwd.cu: warps 0-3 auxiliary, warps 4-15 softmax (three
// per SMSP, the kernel's softmax code on 128x128 TMEM tiles, columns [0, 384)); warp 3 (SMSP 3) either idles, issues
// M=128 N=128 K=16 tcgen05.mma in bursts of 8 into TMEM columns [384, 512) at the kernel's rate (commit + wait per
// burst), or only spins on an mbarrier.  Prints the softmax cycles per tile of each SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_12056_b200/csrc -I tools \
//      tools/mma_interference.cu -o tools/mma_interference.bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "ptx_cta1.cuh"

using namespace spa;
constexpr int ITER = 512;
constexpr int HALF = 64;
constexpr int POLY_FROM = 12;

__device__ __forceinline__ void ex2_poly2(uint64_t X, float &y0, float &y1) {
    float x0, x1;
    ptx::f2unpack(X, x0, x1);
    const uint64_t Xc = ptx::f2pack(fmaxf(x0, -127.f), fmaxf(x1, -127.f));
    const uint64_t T = ptx::fadd2(Xc, ptx::f2pack(12582912.f, 12582912.f));
    const uint64_t F = ptx::fsub2(Xc, ptx::fadd2(T, ptx::f2pack(-12582912.f, -12582912.f)));
    uint64_t P = ptx::ffma2(ptx::f2pack(0.0551716611f, 0.0551716611f), F, ptx::f2pack(0.242611152f, 0.242611152f));
    P = ptx::ffma2(P, F, ptx::f2pack(0.693260968f, 0.693260968f));
    P = ptx::ffma2(P, F, ptx::f2pack(0.999928057f, 0.999928057f));
    float t0, t1;
    ptx::f2unpack(T, t0, t1);
    const float s0 = __int_as_float(__float_as_int(t0) * (1 << 23) + (127 << 23));
    const float s1 = __int_as_float(__float_as_int(t1) * (1 << 23) + (127 << 23));
    ptx::f2unpack(ptx::fmul2(P, ptx::f2pack(s0, s1)), y0, y1);
}

// AUX: 0 = warp 3 idle, 1 = warp 3 issues SS MMAs in bursts of 8, 2 = warp 3 spins on an mbarrier, 3 = TS MMAs
template <int AUX>
__global__ void __launch_bounds__(512, 1) k(unsigned long long *out, float *sink, int mma_batches) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar, never;
    __shared__ volatile int done;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *w = reinterpret_cast<uint32_t *>(smem);
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) w[i] = 0x3c003c00u ^ (i * 2654435761u & 0x007f007fu);
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_init(&never, 1);
        ptx::fence_mbar_init();
        done = 0;
    }
    if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    const uint32_t tm = tbase;
    if (warp >= 4) {
        const int g = (warp - 4) >> 2, wq = warp & 3;
        const uint32_t tS = tm + ((uint32_t)(wq * 32) << 16) + g * 128;
        {
            uint32_t r[32];
            for (int c = 0; c < 4; ++c) {
                for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(((lane * 7 + i * 13 + c) % 29) * 0.37f - 5.f);
                ptx::tmem_st32(tS + c * 32, r);
            }
            ptx::tmem_wait_st();
        }
        const float sl2 = 0.1275174f;
        const uint64_t SL2 = ptx::f2pack(sl2, sl2);
        float mg = 0.f, l = 0.f;
        const uint64_t t0 = clock64();
        for (int it = 0; it < ITER; ++it) {
            float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
            uint32_t kv[HALF];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                uint32_t tv[HALF];
                uint32_t (&sv)[HALF] = r ? kv : tv;
                ptx::tmem_ld_cols<HALF>(tS + HALF * (1 - r), sv);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < HALF; i += 8) {
                    m0 = ptx::fmax3(m0, __uint_as_float(sv[i]), __uint_as_float(sv[i + 1]));
                    m1 = ptx::fmax3(m1, __uint_as_float(sv[i + 2]), __uint_as_float(sv[i + 3]));
                    m2 = ptx::fmax3(m2, __uint_as_float(sv[i + 4]), __uint_as_float(sv[i + 5]));
                    m3 = ptx::fmax3(m3, __uint_as_float(sv[i + 6]), __uint_as_float(sv[i + 7]));
                }
            }
            const float mx = ptx::fmax3(m0, m1, fmaxf(m2, m3)) * sl2;
            const float m = (mx > mg + 8.f) ? mx : mg;
            if (m != mg) { l *= ptx::ex2(mg - m); mg = m; }
            const uint64_t NEGM = ptx::f2pack(-m, -m);
            uint64_t L0 = ptx::f2pack(0.f, 0.f), L1 = L0;
#pragma unroll
            for (int o = 0; o < 2; ++o) {
                const int h = 1 - o;
                uint32_t tv[HALF];
                uint32_t (&sv)[HALF] = o ? tv : kv;
                if (o) {
                    ptx::tmem_ld_cols<HALF>(tS + HALF * h, sv);
                    ptx::tmem_wait_ld();
                }
                uint32_t pk[HALF / 2];
#pragma unroll
                for (int i = 0; i < HALF / 2; ++i) {
                    const int e = 2 * i;
                    const uint64_t X =
                        ptx::ffma2(ptx::f2pack(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), SL2, NEGM);
                    float p0, p1;
                    if ((e & 15) >= POLY_FROM) {
                        ex2_poly2(X, p0, p1);
                    } else {
                        float x0, x1;
                        ptx::f2unpack(X, x0, x1);
                        p0 = ptx::ex2(x0);
                        p1 = ptx::ex2(x1);
                    }
                    if (i & 1) L1 = ptx::fadd2(L1, ptx::f2pack(p0, p1));
                    else L0 = ptx::fadd2(L0, ptx::f2pack(p0, p1));
                    pk[i] = ptx::pack_bf16x2(p0, p1);
                }
                ptx::tmem_st_cols<HALF / 2>(tS + HALF * h, pk);
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                __syncwarp();
            }
            float a0, a1, b0, b1;
            ptx::f2unpack(L0, a0, a1);
            ptx::f2unpack(L1, b0, b1);
            l += (a0 + b0) + (a1 + b1);
        }
        const uint64_t t1 = clock64();
        if (lane == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
        sink[blockIdx.x * blockDim.x + threadIdx.x] = l + mg;
        if (lane == 0) atomicAdd((int *)&done, 1);
    } else if (warp == 3 && AUX == 1) {
        const uint32_t sa = ptx::smem_u32(smem);
        const bool leader = ptx::elect_one();
        int phase = 0;
        for (int b = 0; b < mma_batches && done < 12; ++b) {
            if (leader) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t kk = i & 3;
                    ptx::mma_ss(tm + 384, ptx::smem_desc(sa + kk * 32, 16, 1024, 2),
                                ptx::smem_desc(sa + 32768 + kk * 32, 16, 1024, 2), ptx::idesc_bf16(128, 128, 0, 0),
                                i ? 1u : 0u);
                }
                ptx::mma_commit(&bar);
            }
            __syncwarp();
            ptx::mbar_wait(&bar, phase);
            phase ^= 1;
        }
    } else if (warp == 3 && AUX == 3) {   // TS form (A from TMEM columns [448, 512), like the kernel's PV reading P)
        const uint32_t sa = ptx::smem_u32(smem);
        const bool leader = ptx::elect_one();
        int phase = 0;
        for (int b = 0; b < mma_batches && done < 12; ++b) {
            if (leader) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    ptx::mma_ts(tm + 384, tm + 448 + i * 8, ptx::smem_desc(sa + (i & 3) * 2048, 16, 1024, 2),
                                ptx::idesc_bf16(128, 64, 0, 1), i ? 1u : 0u);
                ptx::mma_commit(&bar);
            }
            __syncwarp();
            ptx::mbar_wait(&bar, phase);
            phase ^= 1;
        }
    } else if (warp == 3 && AUX == 2) {
        while (done < 12) ptx::mbar_try_wait(&never, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tm, 512); }
}

template <int AUX>
void run(const char *name) {
    unsigned long long *d, h[148 * 16];
    float *sink;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&sink, 148 * 512 * 4);
    cudaFuncSetAttribute(k<AUX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
    for (int rep = 0; rep < 2; ++rep) k<AUX><<<148, 512, 70 * 1024>>>(d, sink, 1 << 20);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s err %s\n", name, cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s[4] = {0, 0, 0, 0};
    int n[4] = {0, 0, 0, 0};
    for (int b = 0; b < 148; ++b)
        for (int w = 4; w < 16; ++w) { s[w & 3] += h[b * 16 + w]; ++n[w & 3]; }
    printf("{\"aux\": \"%s\", \"softmax_cycles_per_tile_per_warp\": [%.1f, %.1f, %.1f, %.1f]}\n", name,
           s[0] / n[0] / ITER, s[1] / n[1] / ITER, s[2] / n[2] / ITER, s[3] / n[3] / ITER);
    cudaFree(d);
    cudaFree(sink);
}

int main() {
    run<0>("idle");
    run<1>("mma_bursts_of_8");
    run<2>("spin_try_wait");
    run<3>("mma_ts_bursts_of_8");
    run<0>("idle");
    return 0;
}
