// reshard.cu -- the data-movement kernel of the reshard steps and of the
// loopback transport: a batched strided-run copy.
//
// Every reshard step of the path is a pure permutation made of contiguous runs of g*D*2 bytes
// (one token's heads of one head group, >= 128 B) or whole messages:
//   pack   (seq->head send layout):  send[kh][q][b][t][jj][d] = X[b][t][q*h + kh*g + jj][d]
//   unpack (Psi_g fused gather):     out[b][t][p*h + kh*g + jj][d] = orecv[kh][p][b][t][jj][d]
// (PAPER.md:66 for the all-to-all, PAPER.md:98-101 / 516-578 for Psi.)
// A job enumerates runs with a 4-level index (i3,i2,i1,i0) and byte strides; each thread moves
// one 64-byte quad (4 x 16-B vector loads, then 4 x 16-B stores), so reads and writes are
// coalesced 16-B accesses within runs.  Grid = multiple of the 148 SMs, grid-stride loop.
// The quad -> (run, i0..i3) decomposition uses 32-bit multiply-high division by host-precomputed
// magic numbers (64-bit integer division would make the copy ALU-bound: ~26 % ALU, 34 % of HBM
// peak in profiles/r01_v4/ncu_full_copy_runs.json).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "spa_internal.h"

namespace spa {

namespace {

// n / d for any 32-bit n as (umulhi(n, m) + n) >> l, with l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1
struct FastDiv {
    uint32_t d, m, l;
};
FastDiv make_fastdiv(uint32_t d) {
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    const uint64_t m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;
    return FastDiv{d, (uint32_t)m, l};
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
    return (uint32_t)(((uint64_t)__umulhi(n, f.m) + n) >> f.l);
}

struct JobPack {
    CopyJob job[kMaxCopyJobs];
    long long quad_end[kMaxCopyJobs];  // exclusive prefix sums of quads per job
    FastDiv qpr[kMaxCopyJobs], c3[kMaxCopyJobs], c2[kMaxCopyJobs], c1[kMaxCopyJobs];
    int n;
};

__device__ __forceinline__ uint4 ld_nc(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_na(uint4 *p, const uint4 &v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

__global__ void __launch_bounds__(256) copy_runs_kernel(const __grid_constant__ JobPack jp) {
    const long long total = jp.quad_end[jp.n - 1];
    const long long stride = (long long)gridDim.x * blockDim.x;
    int job = 0;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += stride) {
        while (q >= jp.quad_end[job]) ++job;
        while (job > 0 && q < jp.quad_end[job - 1]) --job;
        const CopyJob &J = jp.job[job];
        const uint32_t local = (uint32_t)(q - (job ? jp.quad_end[job - 1] : 0));   // < 2^32 (host-checked)
        uint32_t run = fdiv(local, jp.qpr[job]);
        const uint32_t qq = local - run * jp.qpr[job].d;
        uint32_t nx = fdiv(run, jp.c3[job]);
        const uint32_t i0 = run - nx * jp.c3[job].d;
        run = nx;
        nx = fdiv(run, jp.c2[job]);
        const uint32_t i1 = run - nx * jp.c2[job].d;
        run = nx;
        const uint32_t i3 = fdiv(run, jp.c1[job]);
        const uint32_t i2 = run - i3 * jp.c1[job].d;
        const uint8_t *s = J.src + i3 * J.src_stride[0] + i2 * J.src_stride[1] + i1 * J.src_stride[2] +
                           i0 * J.src_stride[3] + qq * 64;
        uint8_t *d = J.dst + i3 * J.dst_stride[0] + i2 * J.dst_stride[1] + i1 * J.dst_stride[2] +
                     i0 * J.dst_stride[3] + qq * 64;
        const uint4 *sv = reinterpret_cast<const uint4 *>(s);
        uint4 v0 = ld_nc(sv), v1 = ld_nc(sv + 1), v2 = ld_nc(sv + 2), v3 = ld_nc(sv + 3);
        uint4 *dv = reinterpret_cast<uint4 *>(d);
        st_na(dv, v0);
        st_na(dv + 1, v1);
        st_na(dv + 2, v2);
        st_na(dv + 3, v3);
    }
}

}  // namespace

cudaError_t launch_copy_jobs(const CopyJob *jobs, int n, cudaStream_t st, int *launches) {
    int nl = 0;
    for (int base = 0; base < n; base += kMaxCopyJobs) {
        JobPack jp;
        memset(&jp, 0, sizeof(jp));
        long long acc = 0;
        int m = 0;
        for (int i = base; i < n && m < kMaxCopyJobs; ++i) {
            const CopyJob &J = jobs[i];
            long long runs = J.count[0] * J.count[1] * J.count[2] * J.count[3];
            if (runs <= 0 || J.run_bytes <= 0) continue;
            const long long quads = runs * (J.run_bytes >> 6);
            if (quads >= (1ll << 32)) return cudaErrorInvalidValue;   // 32-bit quad index per job (256 GB)
            jp.job[m] = J;
            jp.qpr[m] = make_fastdiv((uint32_t)(J.run_bytes >> 6));
            jp.c3[m] = make_fastdiv((uint32_t)J.count[3]);
            jp.c2[m] = make_fastdiv((uint32_t)J.count[2]);
            jp.c1[m] = make_fastdiv((uint32_t)J.count[1]);
            acc += quads;
            jp.quad_end[m] = acc;
            ++m;
        }
        if (m == 0) continue;
        jp.n = m;
        // 8 CTAs of 256 threads per SM resident; cap the grid at 2 waves of that, floor at 1 CTA.
        long long ctas = (acc + 255) / 256;
        const long long cap = 148LL * 8 * 2;
        if (ctas > cap) ctas = cap;
        copy_runs_kernel<<<(unsigned)ctas, 256, 0, st>>>(jp);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        ++nl;
    }
    if (launches) *launches += nl;
    return cudaSuccess;
}

}  // namespace spa
