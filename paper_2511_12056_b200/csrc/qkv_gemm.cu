// qkv_gemm.cu -- the QKV projections of a DiT block (Q = X W_Q, K = X W_K, V = X W_V) as a
// persistent tcgen05 GEMM whose epilogue stores straight into the PipeSP send layout (the pack step a1 is fused
// into the projection: the projections overlap the input all-to-alls).
//
//   Y[m, n] = sum_k X[m, k] * Wp[n, k] + bias[n]        m < M (tokens of this rank), n < N, k < K (hidden dim C)
//
// Wp holds one head group's rows of the fused weight in [tensor t][dest rank q][r < g*D] order (packed once per
// plan by spa_plan_pack_qkv_weight), so column n = (t*P + q)*g*D + r lands at
//   dst[t] + q*q_stride + m*row_stride + r       (bf16, RNE from the fp32 accumulator + fp32 bias)
// or, with the direct transport, at peer[q] + off[t] + row'(m)*row_stride + r: destination rank q's receive region over
// peer memory (NVLink), so the projection, the pack and the input all-to-all are one kernel.
// which is send_t[kh][q][b][t][jj][d] for the stage's head group -- or, for a 1-rank plan, the
// plain [B, S, H, D] Q/K/V tensors.
//
// Design (DESIGN.md §5 "QKV projection"): clusters of 2 CTAs act as one tcgen05 CTA pair (cta_group::2): a pair
// tile is 256 rows x 256 columns, each CTA holds its own 128 rows of X and half (128 rows) of the weight tile in
// shared memory (2-SM TMA, 128B swizzle, 64-element K steps, 6-stage ring), the leader's single elected thread
// issues M=256 N=256 K=16 MMAs into a double-buffered fp32 accumulator in TMEM (2 x 256 columns), and four
// epilogue warps per CTA drain one accumulator (tcgen05.ld, bias, bf16, 64-B row segments to global) while the
// MMAs fill the other.  Persistent: the grid is one pair per two SMs (minus SMs left to communication kernels);
// tiles are walked column-fastest so that a wave shares each X tile across the weight's column tiles while the
// weight (<= 19 MB per head group) stays in L2.  Every output element's K reduction runs in the same order in
// every launch, so results are independent of the head-group split.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "ptx.cuh"
#include "spa_internal.h"

namespace spa {

namespace {

constexpr int GM = 128;                  // X rows per CTA (the pair: 256)
constexpr int GN = 256;                  // output columns per pair tile (MMA N); each CTA holds GN/2 weight rows
constexpr int GK = 64;                   // K elements per ring stage (one 128-byte swizzle row)
constexpr int GSTAGES = 6;
constexpr int A_BYTES = GM * GK * 2;     // 16 KB
constexpr int B_BYTES = (GN / 2) * GK * 2;   // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int GTHREADS = 256;            // warp 0 TMA, warp 1 TMEM + MMA, warps 2-3 idle, warps 4-7 epilogue
constexpr int EPI_WARP0 = 4;
constexpr int ACC_COLS = GN;             // fp32 accumulator columns per buffer (two buffers: 512)
constexpr int GSMEM = 1024 + GSTAGES * STAGE_BYTES + 256;
constexpr uint16_t PAIR = 0x3;

struct GemmBars {
    uint64_t full[GSTAGES];    // leader's: TMA bytes of both CTAs for the stage
    uint64_t empty[GSTAGES];   // both CTAs: the MMAs that read the stage completed (multicast commit)
    uint64_t acc_full[2];      // both CTAs: the tile's MMAs into accumulator buffer a completed
    uint64_t acc_empty[2];     // leader's: the 8 epilogue warps of the pair drained buffer a
    uint32_t tmem_base;
};
static_assert(sizeof(GemmBars) <= 256, "barrier block");

__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 2-D TMA load into this CTA's smem, completion counted on the leader CTA's mbarrier (cta_group::2 form).
__device__ __forceinline__ void tma_load_2d_2sm(const CUtensorMap *m, uint32_t bar_cluster_addr, void *dst, int c0,
                                                int c1, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(ptx::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster_addr), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}

__global__ void __launch_bounds__(GTHREADS, 1)
    qkv_gemm_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                    const QkvArgs args) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    GemmBars *bars = reinterpret_cast<GemmBars *>(smem + GSTAGES * STAGE_BYTES);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = ptx::cluster_ctarank();
    const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
    const int nk = (args.K + GK - 1) / GK;

    if (threadIdx.x == 0) {
        for (int i = 0; i < GSTAGES; ++i) {
            ptx::mbar_init(&bars->full[i], 1);
            ptx::mbar_init(&bars->empty[i], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&bars->acc_full[a], 1);
            ptx::mbar_init(&bars->acc_empty[a], 8);   // 4 epilogue warps x 2 CTAs
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmX);
        ptx::prefetch_tmap(&tmW);
    }
    if (warp == 1) {   // same warp id in both CTAs (cta_group::2 allocation)
        ptx::tmem_alloc2(&bars->tmem_base, 2 * ACC_COLS);
        ptx::tmem_relinquish2();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer (both CTAs)
        if (lane == 0) {
            const uint64_t pol_x = policy_evict_normal(), pol_w = ptx::policy_evict_last();
            int it = 0;
            for (int tile = cluster; tile < args.tiles; tile += n_clusters) {
                const int m0 = (tile / args.tiles_n) * (2 * GM) + (int)crank * GM;
                const int n0 = (tile % args.tiles_n) * GN + (int)crank * (GN / 2);
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int slot = it % GSTAGES;
                    ptx::mbar_wait(&bars->empty[slot], ((it / GSTAGES) & 1) ^ 1);
                    uint8_t *st = smem + slot * STAGE_BYTES;
                    const uint32_t bar = ptx::mapa(&bars->full[slot], 0);
                    if (crank == 0) ptx::mbar_arrive_expect_tx(&bars->full[slot], 2 * STAGE_BYTES);
                    tma_load_2d_2sm(&tmX, bar, st, kb * GK, m0, pol_x);
                    tma_load_2d_2sm(&tmW, bar, st + A_BYTES, kb * GK, n0, pol_w);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (leader CTA, one elected lane)
        if (crank == 0) {
            constexpr uint32_t IDESC = ptx::idesc_bf16(2 * GM, GN, 0, 0);
            const uint32_t base = ptx::smem_u32(smem);
            const uint64_t dA = ptx::smem_desc(base, 16, 1024, 2), dB = ptx::smem_desc(base + A_BYTES, 16, 1024, 2);
            const bool leader = ptx::elect_one();
            int it = 0, tcount = 0;
            for (int tile = cluster; tile < args.tiles; tile += n_clusters, ++tcount) {
                const int a = tcount & 1, u = tcount >> 1;
                ptx::mbar_wait(&bars->acc_empty[a], (u & 1) ^ 1);   // the pair's epilogue drained buffer a
                ptx::tc_fence_after();
                const uint32_t d = tmem + a * ACC_COLS;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int slot = it % GSTAGES;
                    ptx::mbar_wait(&bars->full[slot], (it / GSTAGES) & 1);
                    ptx::tc_fence_after();
                    if (leader) {
                        const uint64_t so = (uint64_t)(slot * STAGE_BYTES) >> 4;
#pragma unroll
                        for (int kk = 0; kk < GK / 16; ++kk)
                            ptx::mma_ss2(d, dA + so + ((kk * 32) >> 4), dB + so + ((kk * 32) >> 4), IDESC,
                                         (kb | kk) ? 1u : 0u);
                        ptx::mma_commit2_mc(&bars->empty[slot], PAIR);
                    }
                    __syncwarp();
                }
                if (leader) ptx::mma_commit2_mc(&bars->acc_full[a], PAIR);
                __syncwarp();
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ------------------------------------------------------------ epilogue (both CTAs): TMEM -> bf16 -> global
        const int wq = warp & 3;                       // TMEM lane quarter = this warp's 32 rows
        const int row = wq * 32 + lane;
        int tcount = 0;
        for (int tile = cluster; tile < args.tiles; tile += n_clusters, ++tcount) {
            const int a = tcount & 1, u = tcount >> 1;
            ptx::mbar_wait(&bars->acc_full[a], u & 1);
            ptx::tc_fence_after();
            const long long m = (long long)(tile / args.tiles_n) * (2 * GM) + crank * GM + row;
            const int nt = (tile % args.tiles_n) * GN;
            const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + a * ACC_COLS;
#pragma unroll 1
            for (int j = 0; j < GN / 32; ++j) {
                const int n = nt + j * 32;
                if (n >= args.N) break;                // warp-uniform (N is a multiple of 32)
                uint32_t r[32];
                ptx::tmem_ld32(taddr + j * 32, r);
                ptx::tmem_wait_ld();
                if (m < args.M) {
                    float bv[32];
                    if (args.bias) {
                        const float4 *b4 = reinterpret_cast<const float4 *>(args.bias + n);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float4 t = __ldg(b4 + i);
                            bv[4 * i] = t.x; bv[4 * i + 1] = t.y; bv[4 * i + 2] = t.z; bv[4 * i + 3] = t.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) bv[i] = 0.f;
                    }
                    uint32_t w[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        w[i] = ptx::pack_bf16x2(__uint_as_float(r[2 * i]) + bv[2 * i],
                                                __uint_as_float(r[2 * i + 1]) + bv[2 * i + 1]);
                    const int t = n / args.cols_per_t;
                    const int rem = n - t * args.cols_per_t;
                    const int q = rem / args.cols_per_q;
                    const int rr = rem - q * args.cols_per_q;
                    __nv_bfloat16 *base;
                    long long row = m;
                    if (args.peer[0]) {   // direct: destination rank q's receive region (peer memory)
                        const int bb = m / args.rows_per_b, tt = m - bb * args.rows_per_b;
                        if (t == 0 && args.q_chunks > 1) {   // Q row tt -> its query chunk's stage region
                            const int c = (int)(((long long)(tt + 1) * args.q_chunks - 1) / args.rows_per_b);
                            const int lo = (int)((long long)c * args.rows_per_b / args.q_chunks);
                            base = args.peer[q] + args.q_chunk_off[c];
                            row = (long long)bb * args.q_chunk_rows[c] + (tt - lo);
                        } else {
                            base = args.peer[q] + (t == 0 ? args.off[0] : (t == 1 ? args.off[1] : args.off[2]));
                            row = (long long)bb * args.batch_rows + tt;
                        }
                    } else {
                        base = (t == 0 ? args.dst[0] : (t == 1 ? args.dst[1] : args.dst[2])) + q * args.q_stride;
                    }
                    uint4 *dst = reinterpret_cast<uint4 *>(base + row * args.row_stride + rr);
                    dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                    dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
                    dst[2] = make_uint4(w[8], w[9], w[10], w[11]);
                    dst[3] = make_uint4(w[12], w[13], w[14], w[15]);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(&bars->acc_empty[a], 0));
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();   // no CTA leaves while its peer may still signal its barriers
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc2(tmem, 2 * ACC_COLS);
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D K-major bf16 map over a [rows][K] matrix (row stride ld elements): box 64 x 128, 128-byte swizzle.
bool make_kmajor_map(CUtensorMap *m, const void *base, long long rows, int K, long long ld) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {GK, 128};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t launch_qkv_gemm(const QkvProblem &p, cudaStream_t st) {
    if (p.M <= 0 || p.N <= 0) return cudaSuccess;
    if (p.K <= 0 || p.K % 8 || p.N % 32 || p.cols_per_q % 32 || p.cols_per_t % p.cols_per_q)
        return cudaErrorInvalidValue;
    CUtensorMap mx, mw;
    if (!make_kmajor_map(&mx, p.x, p.M, p.K, p.K) || !make_kmajor_map(&mw, p.w, p.N, p.K, p.K))
        return cudaErrorInvalidValue;
    static std::atomic<uint64_t> attr_done{0};   // per-device smem opt-in (see attn_fwd.cu)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(qkv_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GSMEM);
        if (e != cudaSuccess) return e;
        attr_done.fetch_or(bit, std::memory_order_release);
    }
    int sms = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    QkvArgs a{};
    a.M = p.M; a.N = p.N; a.K = p.K;
    a.tiles_n = (p.N + GN - 1) / GN;
    a.tiles = ((p.M + 2 * GM - 1) / (2 * GM)) * a.tiles_n;
    a.bias = p.bias;
    for (int t = 0; t < 3; ++t) a.dst[t] = reinterpret_cast<__nv_bfloat16 *>(p.dst[t]);
    a.q_stride = p.q_stride; a.row_stride = p.row_stride;
    a.cols_per_t = p.cols_per_t; a.cols_per_q = p.cols_per_q;
    for (int q = 0; q < kMaxDst; ++q) a.peer[q] = reinterpret_cast<__nv_bfloat16 *>(p.peer[q]);
    for (int t = 0; t < 3; ++t) a.off[t] = p.off[t];
    a.rows_per_b = p.rows_per_b > 0 ? p.rows_per_b : 1;
    a.batch_rows = p.batch_rows;
    if (p.q_chunks < 1 || p.q_chunks > kMaxQChunks) return cudaErrorInvalidValue;
    a.q_chunks = p.q_chunks;
    for (int c = 0; c < kMaxQChunks; ++c) { a.q_chunk_off[c] = p.q_chunk_off[c]; a.q_chunk_rows[c] = p.q_chunk_rows[c]; }
    const int usable = sms - (p.reserve_sms > 0 ? p.reserve_sms : 0);
    const int clusters = std::max(1, std::min(a.tiles, usable / 2));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(GTHREADS);
    cfg.dynamicSmemBytes = GSMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, qkv_gemm_kernel, mx, mw, a);
}

}  // namespace spa
