// softmax_microbench.cu -- cycles per 128x128 softmax tile (pass 1 max + pass 2 exp/sum/pack/store)
// from/to TMEM, one thread per row, for several instruction mixes.  Design input for attn_fwd.cu.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_12056_b200/csrc -I tools tools/softmax_microbench.cu -o tools/sm_mb.bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx_cta1.cuh"

using namespace spa;
constexpr int ITER = 256;

__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -125.f);
    const float t = x + 12582912.f;
    const float f = x - (t - 12582912.f);
    float p = fmaf(0.0551716611f, f, 0.242611152f);
    p = fmaf(p, f, 0.693260968f);
    p = fmaf(p, f, 0.999928057f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ void up2(uint64_t r, float &a, float &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
// two exps by the polynomial with packed f32x2 arithmetic
__device__ __forceinline__ void ex2_poly2(float x0, float x1, float &y0, float &y1) {
    x0 = fmaxf(x0, -125.f); x1 = fmaxf(x1, -125.f);
    const uint64_t X = pk2(x0, x1);
    const uint64_t M = pk2(12582912.f, 12582912.f), NM = pk2(-12582912.f, -12582912.f);
    const uint64_t T = fadd2(X, M);
    const uint64_t R = fadd2(T, NM);
    uint64_t F; { float r0, r1; up2(R, r0, r1); F = fadd2(X, pk2(-r0, -r1)); }
    uint64_t P = ffma2(pk2(0.0551716611f, 0.0551716611f), F, pk2(0.242611152f, 0.242611152f));
    P = ffma2(P, F, pk2(0.693260968f, 0.693260968f));
    P = ffma2(P, F, pk2(0.999928057f, 0.999928057f));
    float p0, p1, t0, t1; up2(P, p0, p1); up2(T, t0, t1);
    y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
    y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

template <int VARIANT, int POLY_FROM>
__global__ void __launch_bounds__(256, 1) k(unsigned long long *out, float *sink) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    const uint32_t tS = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
    // fill S with something like scores
    {
        uint32_t r[32];
        for (int c = 0; c < 4; ++c) {
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(((lane * 7 + i * 13 + c) % 29) * 0.1f - 1.4f);
            ptx::tmem_st32(tS + c * 32, r);
        }
        ptx::tmem_wait_st();
    }
    __syncthreads();
    const float sl2 = 0.12752f;
    float m = -INFINITY, l = 0.f;
    uint64_t t0 = clock64();
    for (int it = 0; it < ITER; ++it) {
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            ptx::tmem_ld32(tS + c * 32, r);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                mx0 = fmaxf(mx0, __uint_as_float(r[i])); mx1 = fmaxf(mx1, __uint_as_float(r[i + 1]));
                mx2 = fmaxf(mx2, __uint_as_float(r[i + 2])); mx3 = fmaxf(mx3, __uint_as_float(r[i + 3]));
            }
        }
        const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
        float factor = 1.f;
        if (mx > m + 8.f) { factor = ptx::ex2(m - mx); m = mx; }
        l *= factor;
        float la = 0.f, lb = 0.f;
        uint64_t L = pk2(0.f, 0.f);
        const uint64_t SL2 = pk2(sl2, sl2), NEGM = pk2(-m, -m);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            uint32_t ra[32], rb[32];
            ptx::tmem_ld32(tS + c * 64, ra);
            ptx::tmem_ld32(tS + c * 64 + 32, rb);
            ptx::tmem_wait_ld();
            uint32_t pk[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int e = 2 * i;
                const float s0 = __uint_as_float(e < 32 ? ra[e] : rb[e - 32]);
                const float s1 = __uint_as_float(e + 1 < 32 ? ra[e + 1] : rb[e + 1 - 32]);
                float p0, p1;
                if (VARIANT == 0) {
                    const float x0 = fmaf(s0, sl2, -m), x1 = fmaf(s1, sl2, -m);
                    p0 = ((e & 7) >= POLY_FROM) ? ex2_poly(x0) : ptx::ex2(x0);
                    p1 = (((e + 1) & 7) >= POLY_FROM) ? ex2_poly(x1) : ptx::ex2(x1);
                    la += p0; lb += p1;
                } else {
                    const uint64_t X = ffma2(pk2(s0, s1), SL2, NEGM);
                    float x0, x1; up2(X, x0, x1);
                    if ((e & 7) >= POLY_FROM) ex2_poly2(x0, x1, p0, p1);
                    else { p0 = ptx::ex2(x0); p1 = ptx::ex2(x1); }
                    L = fadd2(L, pk2(p0, p1));
                }
                pk[i] = ptx::pack_bf16x2(p0, p1);
            }
            ptx::tmem_st32(tS + c * 32 + 64, pk);   // keep S intact for the next iteration
            ptx::tmem_wait_st();
        }
        if (VARIANT == 0) l += la + lb;
        else { float a, b; up2(L, a, b); l += a + b; }
    }
    uint64_t t1 = clock64();
    if (lane == 0) out[blockIdx.x * 8 + warp] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = l + m;
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tbase, 512);
}

template <int V, int PF>
void run(const char *name, int nthreads) {
    unsigned long long *d, h[148 * 8]; float *sink;
    cudaMalloc(&d, sizeof(h)); cudaMalloc(&sink, 148 * 256 * 4);
    k<V, PF><<<148, nthreads>>>(d, sink);
    k<V, PF><<<148, nthreads>>>(d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s err %s\n", name, cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0; int n = 0;
    for (int b = 0; b < 148; ++b) for (int w = 0; w < nthreads / 32; ++w) { s += h[b * 8 + w]; ++n; }
    printf("%-36s warps/SMSP=%d  cycles per tile = %7.1f\n", name, nthreads / 128, s / n / ITER);
    cudaFree(d); cudaFree(sink);
}

int main() {
    run<0, 8>("scalar, all MUFU", 128);
    run<0, 5>("scalar, poly 3/8", 128);
    run<0, 4>("scalar, poly 1/2", 128);
    run<1, 8>("packed f32x2, all MUFU", 128);
    run<1, 6>("packed f32x2, poly 1/4", 128);
    run<1, 5>("packed f32x2, poly 3/8", 128);
    run<1, 4>("packed f32x2, poly 1/2", 128);
    run<0, 5>("scalar, poly 3/8 (2 tiles)", 256);
    run<1, 4>("packed, poly 1/2 (2 tiles)", 256);
    run<1, 5>("packed, poly 3/8 (2 tiles)", 256);
    return 0;
}
