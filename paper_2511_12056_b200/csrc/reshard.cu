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
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "spa_internal.h"

namespace spa {

namespace {

struct JobPack {
    CopyJob job[kMaxCopyJobs];
    long long quad_end[kMaxCopyJobs];  // exclusive prefix sums of quads per job
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
        const long long local = q - (job ? jp.quad_end[job - 1] : 0);
        const long long qpr = J.run_bytes >> 6;
        long long run = local / qpr;
        const long long qq = local - run * qpr;
        const long long i0 = run % J.count[3];
        run /= J.count[3];
        const long long i1 = run % J.count[2];
        run /= J.count[2];
        const long long i2 = run % J.count[1];
        const long long i3 = run / J.count[1];
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
            jp.job[m] = J;
            acc += runs * (J.run_bytes >> 6);
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
