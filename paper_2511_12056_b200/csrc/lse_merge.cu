// lse_merge.cu -- combine partial attention results over disjoint key blocks (ring attention, SURVEY.md §8(f)
// f4; R21).  For one output row with partial results O_i = softmax over key block i (normalised)
// and lse_i = ln sum_{t in block i} exp(z_t):
//     O = sum_i exp(lse_i - M) O_i / sum_i exp(lse_i - M),   M = max_i lse_i,
// which is the softmax over the union of the blocks (exact up to rounding).  HBM-bound: n*D*4 bytes read and
// D*2 written per row; one warp per row, float4 loads (D/4 lanes active).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "spa_internal.h"

namespace spa {

namespace {

__global__ void __launch_bounds__(256) lse_merge_kernel(const float *__restrict__ parts, long long part_stride,
                                                        const float *__restrict__ lses, long long lse_stride, int n,
                                                        long long rows, int Sq, int n_heads, int D,
                                                        __nv_bfloat16 *__restrict__ out, long long o_tok_stride,
                                                        long long o_batch_stride) {
    const long long row = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int head = (int)(row % n_heads);
    const long long bs = row / n_heads;
    const int s = (int)(bs % Sq);
    const long long b = bs / Sq;
    float M = -INFINITY;
    for (int i = 0; i < n; ++i) M = fmaxf(M, lses[i * lse_stride + row]);
    const bool active = lane * 4 < D;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float wsum = 0.f;
    if (M != -INFINITY) {
        for (int i = 0; i < n; ++i) {
            const float li = lses[i * lse_stride + row];
            const float w = li == -INFINITY ? 0.f : __expf(li - M);
            wsum += w;
            if (active && w != 0.f) {
                const float4 o = *reinterpret_cast<const float4 *>(parts + i * part_stride + row * D + lane * 4);
                acc.x += w * o.x;
                acc.y += w * o.y;
                acc.z += w * o.z;
                acc.w += w * o.w;
            }
        }
    }
    if (!active) return;
    const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    uint2 v;
    v.x = *reinterpret_cast<uint32_t *>(&lo);
    v.y = *reinterpret_cast<uint32_t *>(&hi);
    *reinterpret_cast<uint2 *>(out + b * o_batch_stride + (long long)s * o_tok_stride + (long long)head * D +
                               lane * 4) = v;
}

}  // namespace

cudaError_t launch_lse_merge(const float *parts, long long part_stride, const float *lses, long long lse_stride,
                             int n, int B, int Sq, int n_heads, int D, void *out, long long o_tok_stride,
                             long long o_batch_stride, cudaStream_t st) {
    const long long rows = (long long)B * Sq * n_heads;
    if (rows == 0 || n <= 0) return cudaSuccess;
    if (D > 128 || D % 4) return cudaErrorInvalidValue;
    const long long blocks = (rows + 7) / 8;
    lse_merge_kernel<<<(unsigned)blocks, 256, 0, st>>>(parts, part_stride, lses, lse_stride, n, rows, Sq, n_heads, D,
                                                       reinterpret_cast<__nv_bfloat16 *>(out), o_tok_stride,
                                                       o_batch_stride);
    return cudaGetLastError();
}

}  // namespace spa
