// lse_merge.cu -- combine partial attention results over disjoint key blocks (ring attention, SURVEY.md §8(f)
// f4; R21).  For one output row with partial results O_i = softmax over key block i (normalised)
// and lse_i = ln sum_{t in block i} exp(z_t):
//     O = sum_i exp(lse_i - M) O_i / sum_i exp(lse_i - M),   M = max_i lse_i,
// which is the softmax over the union of the blocks (exact up to rounding).  HBM-bound: n*D*4 bytes read and
// D*2 written per row.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "spa_internal.h"

namespace spa {

namespace {

// One thread per 4 columns of one row (all lanes busy at D = 96), the row's n lse values read first (L1 broadcast
// across the row's threads), then up to 8 partial float4 loads in flight per thread before any is used: the r01
// one-warp-per-row form waited on each load in turn (long-scoreboard bound, 0.62 of the HBM copy rate).
constexpr int kMergeUnroll = 8;
__global__ void __launch_bounds__(256) lse_merge_kernel(const float *__restrict__ parts, long long part_stride,
                                                        const float *__restrict__ lses, long long lse_stride, int n,
                                                        long long rows, int Sq, int n_heads, int D,
                                                        __nv_bfloat16 *__restrict__ out, long long o_tok_stride,
                                                        long long o_batch_stride) {
    const int q4 = D / 4;   // float4 columns per row
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * q4) return;
    const long long row = idx / q4;
    const int c4 = (int)(idx - row * q4);
    const int head = (int)(row % n_heads);
    const long long bs = row / n_heads;
    const int s = (int)(bs % Sq);
    const long long b = bs / Sq;
    float M = -INFINITY;
    for (int i = 0; i < n; ++i) M = fmaxf(M, __ldg(lses + i * lse_stride + row));
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float wsum = 0.f;
    if (M != -INFINITY) {
        const float4 *p4 = reinterpret_cast<const float4 *>(parts + row * D) + c4;
        const long long ps4 = part_stride / 4;
        for (int i0 = 0; i0 < n; i0 += kMergeUnroll) {
            float4 o[kMergeUnroll];
            float w[kMergeUnroll];
#pragma unroll
            for (int u = 0; u < kMergeUnroll; ++u) {   // every load of the batch issued before the first use
                const int i = i0 + u;
                const float li = i < n ? __ldg(lses + i * lse_stride + row) : -INFINITY;
                w[u] = li == -INFINITY ? 0.f : __expf(li - M);
                o[u] = w[u] != 0.f ? __ldcs(p4 + i * ps4) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < kMergeUnroll; ++u) {
                wsum += w[u];
                acc.x += w[u] * o[u].x;
                acc.y += w[u] * o[u].y;
                acc.z += w[u] * o[u].z;
                acc.w += w[u] * o[u].w;
            }
        }
    }
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    uint2 v;
    v.x = *reinterpret_cast<uint32_t *>(&lo);
    v.y = *reinterpret_cast<uint32_t *>(&hi);
    *reinterpret_cast<uint2 *>(out + b * o_batch_stride + (long long)s * o_tok_stride + (long long)head * D +
                               c4 * 4) = v;
}

}  // namespace

cudaError_t launch_lse_merge(const float *parts, long long part_stride, const float *lses, long long lse_stride,
                             int n, int B, int Sq, int n_heads, int D, void *out, long long o_tok_stride,
                             long long o_batch_stride, cudaStream_t st) {
    const long long rows = (long long)B * Sq * n_heads;
    if (rows == 0 || n <= 0) return cudaSuccess;
    if (D > 128 || D % 4) return cudaErrorInvalidValue;
    const long long blocks = (rows * (D / 4) + 255) / 256;
    lse_merge_kernel<<<(unsigned)blocks, 256, 0, st>>>(parts, part_stride, lses, lse_stride, n, rows, Sq, n_heads, D,
                                                       reinterpret_cast<__nv_bfloat16 *>(out), o_tok_stride,
                                                       o_batch_stride);
    return cudaGetLastError();
}

}  // namespace spa
