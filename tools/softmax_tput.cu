// softmax_tput.cu -- throughput ceiling of the attention kernel's softmax code alone (no MMA, no TMA, no hand-off):
// W softmax warps per SM sub-partition each stream 128x128 tiles through TMEM exactly as attn_fwd.cu's softmax
// warps do (pass 1: two 64-column tcgen05.ld + FMNMX3 max; pass 2: the half still in registers first, FFMA2 scale,
// MUFU.EX2 / FMA-pipe polynomial split by column, FADD2 sums, bf16 pack, tcgen05.st over the scores, wait::st,
// fence, syncwarp).  Prints cycles per tile per SMSP (= per-warp cycles per tile / W): if this is close to the
// kernel's measured period per tile, the softmax instruction stream itself is the limit; if well below, the
// coupling with the MMA pipeline is.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_12056_b200/csrc -I tools \
//      tools/softmax_tput.cu -o tools/softmax_tput.bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "ptx_cta1.cuh"

using namespace spa;
constexpr int ITER = 512;
constexpr int HALF = 64;

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

// MODE 0: the kernel's code; 1: pass 2 only (both halves loaded in pass 2, no pass 1); 2: pass 1 only;
// 3: pass 2 without the polynomial/MUFU (FFMA2 + FADD2 + pack only: the non-exp work); 4: the kernel's arithmetic
// with no TMEM traffic in the loop (scores stay in registers, P folded into a checksum); 5: the kernel with the
// second half's TMEM load issued before the first half is processed; 6: the kernel without the row-sum FADD2s (as if
// the tensor core summed P); 7: 6 with f16x2 MUFU exponentials for the MUFU pairs (x packed to f16x2, P stays f16:
// the exp cost of an f16-P design); 8: single load round (all 128 scores in registers, no reload in pass 2)
template <int MODE, int POLY_FROM, int NT>
__global__ void __launch_bounds__(NT, 1) k(unsigned long long *out, float *sink) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    const int g = warp >> 2, wq = warp & 3;
    const uint32_t tS = tbase + ((uint32_t)(wq * 32) << 16) + g * 128;
    {
        uint32_t r[32];
        for (int c = 0; c < 4; ++c) {
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(((lane * 7 + i * 13 + c) % 29) * 0.37f - 5.f);
            ptx::tmem_st32(tS + c * 32, r);
        }
        ptx::tmem_wait_st();
    }
    __syncthreads();
    const float sl2 = 0.1275174f;
    const uint64_t SL2 = ptx::f2pack(sl2, sl2);
    float mg = 0.f, l = 0.f;
    uint32_t regs[2][HALF], chk = 0;
    if (MODE == 4) {
        ptx::tmem_ld_cols<HALF>(tS, regs[0]);
        ptx::tmem_ld_cols<HALF>(tS + HALF, regs[1]);
        ptx::tmem_wait_ld();
    }
    uint64_t t0 = clock64();
    for (int it = 0; it < ITER; ++it) {
        float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
        uint32_t kv[HALF];
        uint32_t ka[HALF];
        if (MODE == 8) {
            ptx::tmem_ld_cols<HALF>(tS, ka);
            ptx::tmem_ld_cols<HALF>(tS + HALF, kv);
            ptx::tmem_wait_ld();
        }
        if (MODE != 1 && MODE != 3) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                uint32_t tv[HALF];
                uint32_t (&sv)[HALF] = MODE == 4 ? regs[1 - r] : (MODE == 8 ? (r ? kv : ka) : (r ? kv : tv));
                if (MODE != 4 && MODE != 8) {
                    ptx::tmem_ld_cols<HALF>(tS + HALF * (1 - r), sv);
                    ptx::tmem_wait_ld();
                }
#pragma unroll
                for (int i = 0; i < HALF; i += 8) {
                    m0 = ptx::fmax3(m0, __uint_as_float(sv[i]), __uint_as_float(sv[i + 1]));
                    m1 = ptx::fmax3(m1, __uint_as_float(sv[i + 2]), __uint_as_float(sv[i + 3]));
                    m2 = ptx::fmax3(m2, __uint_as_float(sv[i + 4]), __uint_as_float(sv[i + 5]));
                    m3 = ptx::fmax3(m3, __uint_as_float(sv[i + 6]), __uint_as_float(sv[i + 7]));
                }
            }
        }
        const float mx = ptx::fmax3(m0, m1, fmaxf(m2, m3)) * sl2;
        const float m = (mx > mg + 8.f) ? mx : mg;
        if (m != mg) { l *= ptx::ex2(mg - m); mg = m; }
        if (MODE == 2) { l += m; continue; }
        const uint64_t NEGM = ptx::f2pack(-m, -m);
        uint64_t L0 = ptx::f2pack(0.f, 0.f), L1 = L0;
        uint32_t nx[HALF];
        if (MODE == 5) ptx::tmem_ld_cols<HALF>(tS, nx);
#pragma unroll
        for (int o = 0; o < 2; ++o) {
            const int h = 1 - o;   // HALF_ORDER = {1, 0}
            uint32_t tv[HALF];
            const bool load = (o || MODE == 1 || MODE == 3) && MODE != 4 && MODE != 8;
            uint32_t (&sv)[HALF] = MODE == 4 ? regs[h] : (MODE == 8 ? (o ? ka : kv) : ((MODE == 5 && o) ? nx : (load ? tv : kv)));
            if (load) {
                if (MODE != 5) ptx::tmem_ld_cols<HALF>(tS + HALF * h, sv);
                ptx::tmem_wait_ld();
            }
            uint32_t pk[HALF / 2];
#pragma unroll
            for (int i = 0; i < HALF / 2; ++i) {
                const int e = 2 * i;
                const uint64_t X =
                    ptx::ffma2(ptx::f2pack(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), SL2, NEGM);
                float p0, p1;
                if (MODE == 7 && (e & 15) < POLY_FROM) {
                    float x0, x1;
                    ptx::f2unpack(X, x0, x1);
                    uint32_t hx, hy;
                    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hx) : "f"(x1), "f"(x0));
                    asm("ex2.approx.f16x2 %0, %1;" : "=r"(hy) : "r"(hx));
                    pk[i] = hy;
                    continue;
                }
                if (MODE == 3) {
                    ptx::f2unpack(X, p0, p1);
                } else if ((e & 15) >= POLY_FROM) {
                    ex2_poly2(X, p0, p1);
                } else {
                    float x0, x1;
                    ptx::f2unpack(X, x0, x1);
                    p0 = ptx::ex2(x0);
                    p1 = ptx::ex2(x1);
                }
                if (MODE != 6 && MODE != 7) {
                    if (i & 1) L1 = ptx::fadd2(L1, ptx::f2pack(p0, p1));
                    else L0 = ptx::fadd2(L0, ptx::f2pack(p0, p1));
                }
                if (MODE == 7) asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(pk[i]) : "f"(p1), "f"(p0));
                else pk[i] = ptx::pack_bf16x2(p0, p1);
            }
            if (MODE == 4) {
#pragma unroll
                for (int i = 0; i < HALF / 2; ++i) chk ^= pk[i];
            } else {
                ptx::tmem_st_cols<HALF / 2>(tS + HALF * h + 64 * 0, pk);
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
            }
            __syncwarp();
        }
        float a0, a1, b0, b1;
        ptx::f2unpack(L0, a0, a1);
        ptx::f2unpack(L1, b0, b1);
        l += (a0 + b0) + (a1 + b1);
    }
    uint64_t t1 = clock64();
    if (lane == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = l + mg + (float)chk;
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tbase, 512);
}

template <int MODE, int PF, int NT>
void run1(const char *name, int W) {
    unsigned long long *d, h[148 * 16];
    float *sink;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&sink, 148 * 512 * 4);
    k<MODE, PF, NT><<<148, 128 * W>>>(d, sink);
    k<MODE, PF, NT><<<148, 128 * W>>>(d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s err %s\n", name, cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    int n = 0;
    for (int b = 0; b < 148; ++b)
        for (int w = 0; w < 4 * W; ++w) { s += h[b * 16 + w]; ++n; }
    const double per_warp = s / n / ITER;
    printf("{\"mode\": \"%s\", \"poly_from\": %d, \"warps_per_smsp\": %d, \"cycles_per_tile_per_warp\": %.1f, "
           "\"cycles_per_tile_per_smsp\": %.1f}\n", name, PF, W, per_warp, per_warp / W);
    cudaFree(d);
    cudaFree(sink);
}

template <int MODE, int PF>
void run(const char *name, int W) {
    if (W <= 3) run1<MODE, PF, 384>(name, W);
    else run1<MODE, PF, 512>(name, W);
}

int main() {
    for (int W = 1; W <= 3; ++W) {
        run<8, 12>("one_load_round", W);
        run<8, 10>("one_load_round", W);
        run<0, 12>("kernel", W);
    }
    for (int W = 3; W <= 3; ++W) {
        run<6, 12>("no_rowsum", W);
        run<6, 10>("no_rowsum", W);
        run<6, 8>("no_rowsum", W);
        run<7, 16>("f16_mufu_no_rowsum", W);
        run<7, 12>("f16_mufu_no_rowsum", W);
        run<7, 8>("f16_mufu_no_rowsum", W);
        run<0, 12>("kernel", W);
    }
    for (int W = 1; W <= 4; ++W) {
        run<0, 14>("kernel", W);
        run<0, 12>("kernel", W);
        run<0, 10>("kernel", W);
        run<0, 8>("kernel", W);
        run<0, 16>("kernel", W);
        run<1, 12>("pass2_only", W);
        run<2, 12>("pass1_only", W);
        run<3, 12>("no_exp", W);
        run<4, 12>("no_tmem", W);
        run<4, 16>("no_tmem", W);
        run<5, 12>("prefetch", W);
    }
    return 0;
}
