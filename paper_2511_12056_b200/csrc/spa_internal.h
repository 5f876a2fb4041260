// spa_internal.h -- internal types shared by the library's translation units.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace spa {

constexpr int kMaxDst = 16;   // ranks one attention launch can scatter its output rows to
constexpr int kMaxQChunks = 32;   // query chunks per head group the direct projection GEMM can address

// Attention problem for one launch (a head group of one stage, or a whole single-GPU layer).
// Element (b, s, j, d) of q is at q + b*q_batch_stride + s*q_tok_stride + j*D + d (elements).
struct AttnProblem {
    const void *q, *k, *v;
    void *o;
    int B, Sq, Skv, n_heads, D;
    long long q_tok_stride, q_batch_stride;
    long long kv_tok_stride, kv_batch_stride;
    long long o_tok_stride, o_batch_stride;
    const int32_t *kv_len = nullptr;   // key padding: device int32 [B], keys t >= kv_len[b] masked (NULL: none)
    int kv_offset = 0;                 // global position of this launch's key 0 (ring blocks): t masked iff
                                       // t + kv_offset >= kv_len[b]
    void *o32 = nullptr;               // non-NULL: fp32 output instead of o (same element strides)
    float *lse = nullptr;              // non-NULL: per-row log-sum-exp, [B][Sq][n_heads] contiguous
    // Scattered output (direct transport): n_dst > 0 -> query rows [row_begin[i], row_begin[i+1]) go
    // to dst[i] + b*dst_batch_stride[i] + (s - row_begin[i])*o_tok_stride + j*D (o is unused); row_begin has
    // n_dst + 1 entries.
    int n_dst = 0;
    int row_begin[kMaxDst + 1] = {};
    void *dst[kMaxDst] = {};
    long long dst_batch_stride[kMaxDst] = {};
};

// Kernel-side arguments (tensor maps travel separately as __grid_constant__ parameters).
struct AttnArgs {
    __nv_bfloat16 *O;
    long long o_tok_stride, o_batch_stride;
    int Sq, Skv;
    float scale_log2;
    const int32_t *kv_len;   // NULL or device [B]
    int kv_offset;
    float *O32;              // NULL or fp32 output
    float *lse;              // NULL or [B][Sq][lse_heads]
    int lse_heads;
    int n_dst;               // > 0: scattered output (see AttnProblem)
    int row_begin[kMaxDst + 1];
    __nv_bfloat16 *dst[kMaxDst];
    long long dst_batch_stride[kMaxDst];
};

// out[b, s, j, :] = sum_i w_i O_i[b, s, j, :] / sum_i w_i, w_i = exp(lse_i - max_i lse_i), over n partial results
// O_i (fp32, [B][Sq][n_heads][D] contiguous, at parts + i*part_stride elements) with lse_i ([B][Sq][n_heads] at
// lses + i*lse_stride); out bf16 with token / batch strides (elements).  Rows whose every lse is -inf are 0.
cudaError_t launch_lse_merge(const float *parts, long long part_stride, const float *lses, long long lse_stride,
                             int n, int B, int Sq, int n_heads, int D, void *out, long long o_tok_stride,
                             long long o_batch_stride, cudaStream_t st);

cudaError_t launch_attention(const AttnProblem &p, cudaStream_t st);

// QKV projection GEMM (qkv_gemm.cu): Y[m, n] = sum_k x[m, k] w[n, k] + bias[n] for
// m < M, n < N, k < K (x [M][K], w [N][K] bf16 row-major, bias fp32 [N] or NULL); column n = (t*Q + q)*cols_per_q
// + r (t < 3, cols_per_t = Q*cols_per_q) is stored as bf16 at dst[t] + q*q_stride + m*row_stride + r (elements).
// N, cols_per_q multiples of 32; K multiple of 8; reserve_sms SMs are left free (communication kernels).
struct QkvProblem {
    const void *x, *w;
    const float *bias;
    int M, N, K;
    void *dst[3];
    long long q_stride, row_stride;
    int cols_per_t, cols_per_q;
    int reserve_sms;
    // Direct transport (peer[0] != NULL; SURVEY f1 for the projections): column block q of tensor t goes straight into
    // destination rank q's receive region, peer[q] + off[t] + row'*row_stride + r (elements), with the batch remap
    // row' = (m / rows_per_b) * batch_rows + m % rows_per_b (this source's rows of batch entry b inside the owner's
    // [b][S] rows); dst / q_stride are then unused.
    void *peer[kMaxDst] = {};
    long long off[3] = {};
    int rows_per_b = 1, batch_rows = 1;
    // Query chunks (C > 1): Q row t of this source lies in chunk c = ((t+1)*C - 1) / rows_per_b, i.e. rows
    // [c*rows_per_b/C, (c+1)*rows_per_b/C), and goes to q_chunk_off[c] + (b*q_chunk_rows[c] + t - first row of c)
    // (elements, relative to peer[q]); off[0] and batch_rows are then not used for Q.
    int q_chunks = 1;
    long long q_chunk_off[kMaxQChunks] = {};
    int q_chunk_rows[kMaxQChunks] = {};
};
struct QkvArgs {
    int M, N, K, tiles_n, tiles;
    const float *bias;
    __nv_bfloat16 *dst[3];
    long long q_stride, row_stride;
    int cols_per_t, cols_per_q;
    __nv_bfloat16 *peer[kMaxDst];
    long long off[3];
    int rows_per_b, batch_rows;
    int q_chunks;
    long long q_chunk_off[kMaxQChunks];
    int q_chunk_rows[kMaxQChunks];
};
cudaError_t launch_qkv_gemm(const QkvProblem &p, cudaStream_t st);

// Strided run copy: for (i3,i2,i1,i0) < count: copy run_bytes from
// src + sum(i*src_stride) to dst + sum(i*dst_stride).  run_bytes % 64 == 0, 16-B aligned.
struct CopyJob {
    const uint8_t *src;
    uint8_t *dst;
    long long count[4];
    long long src_stride[4], dst_stride[4];
    long long run_bytes;
};
constexpr int kMaxCopyJobs = 32;
// Launches ceil(n / kMaxCopyJobs) kernels; returns number launched via *launches.
cudaError_t launch_copy_jobs(const CopyJob *jobs, int n, cudaStream_t st, int *launches);

}  // namespace spa
