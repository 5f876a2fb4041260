// attn_fwd.cu -- bf16 flash attention forward for sm_100a on tcgen05 / TMEM / TMA.
//
// Computes, per (batch b, head j, query row s):
//     o[b,s,j,:] = softmax_t( q[b,s,j,:] . k[b,t,j,:] / sqrt(D) ) v[b,t,j,:]
// which is Alg. 1 line 3 `attention(Q[:,j],K[:,j],V[:,j])` for a
// group of heads; the scale 1/sqrt(D) is the north star's (R1).
//
// Design (DESIGN.md §Kernels / attention):
//   * one CTA = 2 query tiles of 128 rows (256 rows) of one (b, head); 12 warps:
//       warp 0       TMA producer: Q0,Q1 once, then K_j, V_j through an NS-slot smem ring
//       warp 1       TMEM allocator + tcgen05.mma issuer (one elected lane)
//       warps 4..7   softmax / correction / epilogue of query tile 0 (one thread per row)
//       warps 8..11  same for query tile 1
//   * S_t = Q_t K_j^T   : tcgen05.mma SS, M=128 N=128, fp32 accumulator in TMEM cols [128t, 128t+128)
//   * P_t (bf16)        : written by the softmax warps back into TMEM over S_t's first 64 columns
//   * O_t += P_t V_j    : tcgen05.mma TS (A = P from TMEM, B = V from smem, MN-major), O_t in TMEM
//   * issue order S0(j), S1(j) ... PV0(j-1), S0(j+1), PV1(j-1), S1(j+1) ping-pongs the tensor core
//     between the two tiles so one tile's softmax overlaps the other tile's MMAs.
//   * online softmax in fp32, base-2 with log2(e)/sqrt(D) folded into one FFMA; the running max
//     is only raised when it grows by more than 2^8 (conditional rescale, exact in the end
//     because the final 1/l uses the same max).  The decision is per row, so a row's result
//     does not depend on which other rows share its tile (bit-identical across stage splits).
//   * keys >= Skv (ragged tail, TMA zero-filled) get score -inf; query rows >= Sq are not stored.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <type_traits>

#include "ptx.cuh"
#include "spa_internal.h"

namespace spa {

namespace {

constexpr int BM = 128;        // query rows per tile (MMA M)
constexpr int BN = 128;        // keys per tile (MMA N of QK^T, K of PV)
// warps: 0 TMA producer, 1 MMA issuer of query tile 0, 2 MMA issuer of tile 1,
// 3..6 softmax/epilogue of tile 0, 7..10 softmax/epilogue of tile 1 (warp w owns TMEM lanes 32*(w%4)..+31).
constexpr int NUM_WARPS = 11;
constexpr int NUM_THREADS = NUM_WARPS * 32;
constexpr int SOFTMAX_WARP0 = 3;
constexpr float RESCALE_TAU = 8.0f;  // log2 domain: raise the running max only if it grows by > 2^8

#ifdef SPA_ATTN_TRACE
// Debug timeline of CTA (0,0,0): slot[j][e] = clock64 at event e of KV iteration j (tools/attn_trace.py).
__device__ unsigned long long g_trace[256][16];
#define TRACE(j, e)                                                                  \
    do {                                                                             \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 256)      \
            g_trace[(j)][(e)] = clock64();                                           \
    } while (0)
#else
#define TRACE(j, e) do {} while (0)
#endif

template <int D>
struct Cfg {
    static_assert(D == 64 || D == 96 || D == 128, "D in {64, 96, 128}");
    // Q/K tiles (K-major operands): 64-column 128B-swizzled chunks + (D=96) one 32-column 64B-swizzled chunk.
    static constexpr int N128 = D / 64;                  // 1, 1, 2
    static constexpr int N64 = (D % 64) ? 1 : 0;         // 0, 1, 0
    static constexpr int NCHUNK = N128 + N64;
    // V tiles (MN-major B operand of PV, N = D in ONE instruction): D=64/128 -> 64-column SW128 atoms,
    // D=96 -> three 32-column SW64 atoms; LBO = distance between atoms along N.
    static constexpr bool V_SW64 = (D == 96);
    static constexpr int V_ATOM_COLS = V_SW64 ? 32 : 64;
    static constexpr int V_ATOMS = D / V_ATOM_COLS;
    static constexpr int V_ATOM_BYTES = BM * V_ATOM_COLS * 2;
    static constexpr int TILE_BYTES = BM * D * 2;
    static constexpr int NS = (D == 64) ? 8 : (D == 96 ? 6 : 4);   // K/V ring slots
    static constexpr int SMEM_TILES = 2 + NS;
    static constexpr int BAR_BYTES = 256;
    static constexpr int SMEM_BYTES = 1024 /*align slack*/ + SMEM_TILES * TILE_BYTES + BAR_BYTES;
    static constexpr uint32_t TMEM_COLS = 512;           // S0 | S1 | O0 | O1 (128 columns each)
    // exp2 split between MUFU and an FMA-pipe polynomial: columns with (i & 7) >= POLY_FROM use the polynomial.
    static constexpr int POLY_FROM = 5;                    // 3/8 of the elements (tools/softmax_microbench.cu)
};

__device__ __forceinline__ int chunk_off(int c) { return c * (BM * 128); }  // Q/K chunk c byte offset in a tile

struct SmemBars {
    uint64_t q_full;
    uint64_t kv_full[8];
    uint64_t kv_empty[8];
    uint64_t s_full[2];
    uint64_t p_full[2][2];   // [tile][half]: P columns of keys 0..63 / 64..127 written
    uint64_t o_full[2];
    uint32_t tmem_base;
};

// 2^x on the FMA pipe: x = n + f (n = round(x), |f| <= 1/2), 2^f by a degree-3 fit (max rel err 7.5e-5,
// far below the bf16 rounding of P), 2^n by adding n to the exponent field.  x is clamped at -125 so the
// result stays a normal number (p >= 0.7 has exponent >= 126).
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -125.f);
    const float t = x + 12582912.f;                      // 1.5 * 2^23: t's low mantissa bits hold round(x)
    const float f = x - (t - 12582912.f);
    float p = fmaf(0.0551716611f, f, 0.242611152f);
    p = fmaf(p, f, 0.693260968f);
    p = fmaf(p, f, 0.999928057f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int D>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQa, const __grid_constant__ CUtensorMap tmQb,
                    const __grid_constant__ CUtensorMap tmKa, const __grid_constant__ CUtensorMap tmKb,
                    const __grid_constant__ CUtensorMap tmVa, const __grid_constant__ CUtensorMap tmVb,
                    const AttnArgs args) {
    using C = Cfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sQ = smem;                               // 2 tiles
    uint8_t *sKV = smem + 2 * C::TILE_BYTES;          // NS tiles
    SmemBars *bars = reinterpret_cast<SmemBars *>(smem + C::SMEM_TILES * C::TILE_BYTES);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int tile2 = blockIdx.x;     // 256-row query block
    const int head = blockIdx.y;
    const int b = blockIdx.z;
    const int n_kv = (args.Skv + BN - 1) / BN;

    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars->q_full, 1);
        for (int i = 0; i < C::NS; ++i) {
            ptx::mbar_init(&bars->kv_full[i], 1);
            ptx::mbar_init(&bars->kv_empty[i], 2);   // released by both tiles' MMA issuers
        }
        for (int t = 0; t < 2; ++t) {
            ptx::mbar_init(&bars->s_full[t], 1);
            ptx::mbar_init(&bars->p_full[t][0], 4);   // one arrival per softmax warp
            ptx::mbar_init(&bars->p_full[t][1], 4);
            ptx::mbar_init(&bars->o_full[t], 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmQa); ptx::prefetch_tmap(&tmKa); ptx::prefetch_tmap(&tmVa);
        if (C::N64) { ptx::prefetch_tmap(&tmQb); ptx::prefetch_tmap(&tmKb); ptx::prefetch_tmap(&tmVb); }
    }
    if (warp == 1) {
        ptx::tmem_alloc(&bars->tmem_base, C::TMEM_COLS);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        const uint64_t pol_q = ptx::policy_evict_first();
        const uint64_t pol_kv = ptx::policy_evict_last();
        // Q/K style (K-major) tile: chunk 0 = cols 0..63 (SW128); chunk 1 = cols 64.. (SW128 or SW64)
        auto load_qk = [&](const CUtensorMap *m64, const CUtensorMap *m32, uint64_t *bar, uint8_t *dst, int row,
                           uint64_t pol) {
            ptx::tma_load_4d(m64, bar, dst, 0, head, row, b, pol);
            if (C::N128 == 2) ptx::tma_load_4d(m64, bar, dst + chunk_off(1), 64, head, row, b, pol);
            if (C::N64) ptx::tma_load_4d(m32, bar, dst + chunk_off(1), 64, head, row, b, pol);
        };
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(&bars->q_full, 2 * C::TILE_BYTES);
            for (int t = 0; t < 2; ++t)
                load_qk(&tmQa, &tmQb, &bars->q_full, sQ + t * C::TILE_BYTES, tile2 * 2 * BM + t * BM, pol_q);
        }
        for (int i = 0; i < 2 * n_kv; ++i) {
            const int slot = i % C::NS;
            const uint32_t use = i / C::NS;
            ptx::mbar_wait(&bars->kv_empty[slot], (use & 1) ^ 1);
            if (lane == 0) TRACE(i >> 1, 14 + (i & 1));
            if (lane == 0) {
                const int j = i >> 1;
                uint8_t *dst = sKV + slot * C::TILE_BYTES;
                ptx::mbar_arrive_expect_tx(&bars->kv_full[slot], C::TILE_BYTES);
                if (i & 1) {   // V_j: D/V_ATOM_COLS atoms
                    const CUtensorMap *mv = C::V_SW64 ? &tmVb : &tmVa;
#pragma unroll
                    for (int a = 0; a < C::V_ATOMS; ++a)
                        ptx::tma_load_4d(mv, &bars->kv_full[slot], dst + a * C::V_ATOM_BYTES, a * C::V_ATOM_COLS,
                                         head, j * BN, b, pol_kv);
                } else {       // K_j
                    load_qk(&tmKa, &tmKb, &bars->kv_full[slot], dst, j * BN, pol_kv);
                }
            }
            __syncwarp();
        }
    } else if (warp == 1 || warp == 2) {
        // ------------------------------------------------------------ MMA issuer of query tile t
        // One issuer per tile: each tile's chain S_t(j) -> softmax_t(j) -> PV_t(j) -> S_t(j+1) advances on
        // its own, and the tensor core interleaves the two chains (in-order per issuing thread, which
        // is what the S/P aliasing in TMEM needs).  Every K/V slot is released by both issuers.
        const int t = warp - 1;
        constexpr uint32_t IDESC_QK = ptx::idesc_bf16(BM, BN, 0, 0);
        constexpr uint32_t IDESC_PV = ptx::idesc_bf16(BM, D, 0, 1);
        const uint32_t qa = ptx::smem_u32(sQ) + t * C::TILE_BYTES;
        const uint32_t sKV_addr = ptx::smem_u32(sKV);
        const uint32_t tS = tmem + t * 128;
        const uint32_t tO = tmem + 256 + t * 128;

        // S_t = Q_t K^T over D: K-major A (Q) and B (K); 16-element k-steps inside each swizzle chunk.
        auto issue_qk = [&](int slot) {
            const uint32_t kb = sKV_addr + slot * C::TILE_BYTES;
            uint32_t acc = 0;
#pragma unroll
            for (int c = 0; c < C::NCHUNK; ++c) {
                const bool sw64 = (c >= C::N128);
                const uint32_t layout = sw64 ? 4u : 2u;
                const uint32_t sbo = sw64 ? 512u : 1024u;
                const int ksteps = sw64 ? 2 : 4;
#pragma unroll
                for (int kk = 0; kk < ksteps; ++kk) {
                    const uint64_t ad = ptx::smem_desc(qa + chunk_off(c) + kk * 32, 16, sbo, layout);
                    const uint64_t bd = ptx::smem_desc(kb + chunk_off(c) + kk * 32, 16, sbo, layout);
                    ptx::mma_ss(tS, ad, bd, IDESC_QK, acc);
                    acc = 1;
                }
            }
        };
        // O_t (+)= P_t V for key steps [k0, k1): A = P from TMEM (8 columns per 16 keys), B = V (N = D).
        auto issue_pv = [&](int slot, uint32_t accum, int k0, int k1) {
            const uint32_t vb = sKV_addr + slot * C::TILE_BYTES;
            constexpr uint32_t rowb = C::V_ATOM_COLS * 2;
#pragma unroll
            for (int kk = k0; kk < k1; ++kk) {
                const uint64_t bd = ptx::smem_desc(vb + kk * 16 * rowb, C::V_ATOM_BYTES, 8 * rowb, C::V_SW64 ? 4u : 2u);
                ptx::mma_ts(tO, tS + kk * 8, bd, IDESC_PV, (accum | kk) ? 1u : 0u);
            }
        };

        ptx::mbar_wait(&bars->q_full, 0);
        ptx::mbar_wait(&bars->kv_full[0], 0);
        ptx::tc_fence_after();
        if (lane == 0) {
            issue_qk(0);
            ptx::mma_commit(&bars->s_full[t]);
            ptx::mma_commit(&bars->kv_empty[0]);
        }
        __syncwarp();
        for (int j = 0; j < n_kv; ++j) {
            const int iV = 2 * j + 1, slotV = iV % C::NS;
            const int iK = 2 * j + 2, slotK = iK % C::NS;
            const bool has_k = j + 1 < n_kv;
            const uint32_t accum = j > 0 ? 1u : 0u;
            ptx::mbar_wait(&bars->kv_full[slotV], (iV / C::NS) & 1);
            if (lane == 0 && t == 0) TRACE(j, 0);
            ptx::mbar_wait(&bars->p_full[t][0], j & 1);      // keys 0..63 of P_t(j)
            ptx::tc_fence_after();
            if (lane == 0) {
                TRACE(j, 1 + t);
                issue_pv(slotV, accum, 0, BN / 32);
            }
            __syncwarp();
            if (has_k) ptx::mbar_wait(&bars->kv_full[slotK], (iK / C::NS) & 1);
            ptx::mbar_wait(&bars->p_full[t][1], j & 1);      // keys 64..127
            ptx::tc_fence_after();
            if (lane == 0) {
                issue_pv(slotV, accum, BN / 32, BN / 16);
                ptx::mma_commit(&bars->kv_empty[slotV]);
                if (has_k) {
                    issue_qk(slotK);
                    ptx::mma_commit(&bars->s_full[t]);
                    ptx::mma_commit(&bars->kv_empty[slotK]);
                } else {
                    ptx::mma_commit(&bars->o_full[t]);
                }
            }
            __syncwarp();
        }
    } else if (warp >= SOFTMAX_WARP0) {
        // ------------------------------------------------------------ softmax / correction / epilogue
        const int t = (warp - SOFTMAX_WARP0) >> 2;     // query tile 0 or 1
        const int wq = warp & 3;                       // TMEM lane quarter this warp may access
        const int row = wq * 32 + lane;                // row within the tile
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_base + t * 128;
        const uint32_t tO = tmem + lane_base + 256 + t * 128;
        const float sl2 = args.scale_log2;
                const int last_valid = args.Skv - (n_kv - 1) * BN;   // valid keys in the last tile (1..128)

        float m = -INFINITY;   // running max, already scaled to the log2 domain
        float l = 0.f;         // running sum of p (fp32)
        // one KV iteration; MASK instantiates the ragged last tile separately (keys >= Skv -> -inf), so the
        // common path carries no masking code
        auto step = [&](const int j, const bool MASK) {
            const bool tr = (lane == 0 && wq == 0);
            if (tr) TRACE(j, 3 + 5 * t);
            ptx::mbar_wait(&bars->s_full[t], j & 1);
            ptx::tc_fence_after();
            if (tr) TRACE(j, 4 + 5 * t);
            // pass 1: row max over all 128 keys (4 TMEM loads, one wait)
            float mx0, mx1, mx2, mx3;
            {
                uint32_t sv[BN / 32][32];
#pragma unroll
                for (int c = 0; c < BN / 32; ++c) ptx::tmem_ld32(tS + c * 32, sv[c]);
                ptx::tmem_wait_ld();
                if (tr) TRACE(j, 5 + 5 * t);
                if (MASK) {
#pragma unroll
                    for (int i = 0; i < BN; ++i)
                        if (i >= last_valid) sv[i >> 5][i & 31] = __float_as_uint(-INFINITY);
                }
                mx0 = __uint_as_float(sv[0][0]); mx1 = __uint_as_float(sv[0][1]);
                mx2 = __uint_as_float(sv[0][2]); mx3 = __uint_as_float(sv[0][3]);
#pragma unroll
                for (int i = 4; i < BN; i += 4) {
                    mx0 = fmaxf(mx0, __uint_as_float(sv[i >> 5][i & 31]));
                    mx1 = fmaxf(mx1, __uint_as_float(sv[i >> 5][(i + 1) & 31]));
                    mx2 = fmaxf(mx2, __uint_as_float(sv[i >> 5][(i + 2) & 31]));
                    mx3 = fmaxf(mx3, __uint_as_float(sv[i >> 5][(i + 3) & 31]));
                }
            }
            const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
            float factor = 1.f;
            if (mx > m + RESCALE_TAU) {            // also true on the first tile (m = -inf)
                factor = ptx::ex2(m - mx);         // 0 on the first tile
                m = mx;
            }
            l *= factor;
            // Correction of O_t before any PV of this iteration is issued (the previous PV of this tile
            // completed before s_full fired).  Rows that keep their max multiply by exactly 1.
            const bool need = (j > 0) && (factor != 1.f);
            if (__any_sync(0xffffffffu, need)) {
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    uint32_t r[32];
                    ptx::tmem_ld32(tO + c * 32, r);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * factor);
                    ptx::tmem_st32(tO + c * 32, r);
                }
            }
            // P = exp2(s*sl2 - m) in f32x2 pairs (MUFU or FMA-pipe polynomial by column), rounded to bf16
            // pairs, written over S's first 64 columns in two halves (keys 0..63, 64..127), each
            // released to the MMA issuer as soon as it is in TMEM.
            // pass 2 (per half of 64 keys): reload S from TMEM, P = exp2(s*sl2 - m) (MUFU or FMA-pipe
            // polynomial by column), bf16 pairs written over S's first 64 columns, half released to the
            // MMA issuer as soon as it is in TMEM.  Keeping only 64 scores live avoids register spills.
            float la = 0.f, lb = 0.f;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t sa[32], sb[32];
                ptx::tmem_ld32(tS + c * 64, sa);
                ptx::tmem_ld32(tS + c * 64 + 32, sb);
                ptx::tmem_wait_ld();
                if (MASK) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        if (c * 64 + i >= last_valid) sa[i] = __float_as_uint(-INFINITY);
                        if (c * 64 + 32 + i >= last_valid) sb[i] = __float_as_uint(-INFINITY);
                    }
                }
                uint32_t pk[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int e = 2 * i;   // key index within the half
                    const float s0 = __uint_as_float(e < 32 ? sa[e] : sb[e - 32]);
                    const float s1 = __uint_as_float(e + 1 < 32 ? sa[e + 1] : sb[e + 1 - 32]);
                    const float x0 = fmaf(s0, sl2, -m);
                    const float x1 = fmaf(s1, sl2, -m);
                    const float p0 = ((e & 7) >= C::POLY_FROM) ? ex2_poly(x0) : ptx::ex2(x0);
                    const float p1 = (((e + 1) & 7) >= C::POLY_FROM) ? ex2_poly(x1) : ptx::ex2(x1);
                    la += p0;
                    lb += p1;
                    pk[i] = ptx::pack_bf16x2(p0, p1);
                }
                ptx::tmem_st32(tS + c * 32, pk);
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&bars->p_full[t][c]);
            }
            l += la + lb;
            if (tr) TRACE(j, 6 + 5 * t);
            if (tr) TRACE(j, 7 + 5 * t);
        };
        for (int j = 0; j < n_kv; ++j) step(j, j == n_kv - 1 && last_valid < BN);
        // ------------------------------------------------------------ epilogue: O / l -> bf16 -> global
        ptx::mbar_wait(&bars->o_full[t], 0);
        ptx::tc_fence_after();
        const float inv_l = 1.f / l;
        const long long srow = (long long)tile2 * 2 * BM + t * BM + row;
        const bool valid = srow < args.Sq;
        __nv_bfloat16 *orow = args.O + (long long)b * args.o_batch_stride + srow * args.o_tok_stride +
                              (long long)head * D;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            ptx::tmem_ld32(tO + c * 32, r);
            ptx::tmem_wait_ld();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
                pk[i] = ptx::pack_bf16x2(__uint_as_float(r[2 * i]) * inv_l, __uint_as_float(r[2 * i + 1]) * inv_l);
            if (valid) {
                uint4 *dst = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                for (int v = 0; v < 4; ++v) dst[v] = make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// ------------------------------------------------------------------ host side
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
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

// 4-D map over a [B][S][heads][D] bf16 view: dims (D, heads, S, B), box (box_d, 1, 128, 1).
bool make_map(CUtensorMap *m, const void *base, int D, int heads, int S, int B, long long tok_stride,
              long long batch_stride, int box_d, bool sw64) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)heads, (cuuint64_t)S, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)tok_stride * 2, (cuuint64_t)batch_stride * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_d, 1, (cuuint32_t)BM, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sw64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int D>
cudaError_t launch_d(const AttnProblem &p, cudaStream_t st) {
    using C = Cfg<D>;
    // m[0]/m[2]: Q/K 64-col SW128 boxes; m[1]/m[3]: Q/K 32-col SW64 boxes (D=96 tail chunk);
    // m[4]: V 64-col SW128 boxes (D=64/128); m[5]: V 32-col SW64 boxes (D=96).
    CUtensorMap m[6];
    bool ok = make_map(&m[0], p.q, D, p.n_heads, p.Sq, p.B, p.q_tok_stride, p.q_batch_stride, 64, false) &&
              make_map(&m[2], p.k, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, 64, false);
    if (ok && C::N64)
        ok = make_map(&m[1], p.q, D, p.n_heads, p.Sq, p.B, p.q_tok_stride, p.q_batch_stride, 32, true) &&
             make_map(&m[3], p.k, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, 32, true);
    else {
        m[1] = m[0];
        m[3] = m[2];
    }
    if (ok) ok = C::V_SW64 ? make_map(&m[5], p.v, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, 32, true)
                           : make_map(&m[4], p.v, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, 64, false);
    if (C::V_SW64) m[4] = m[5];
    else m[5] = m[4];
    if (!ok) return cudaErrorInvalidValue;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    AttnArgs a;
    a.O = reinterpret_cast<__nv_bfloat16 *>(p.o);
    a.o_tok_stride = p.o_tok_stride;
    a.o_batch_stride = p.o_batch_stride;
    a.Sq = p.Sq;
    a.Skv = p.Skv;
    a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
    dim3 grid((p.Sq + 2 * BM - 1) / (2 * BM), p.n_heads, p.B);
    attn_fwd_kernel<D><<<grid, NUM_THREADS, C::SMEM_BYTES, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], a);
    return cudaGetLastError();
}

}  // namespace

#ifdef SPA_ATTN_TRACE
extern "C" int spa_debug_read_trace(unsigned long long *out) {
    return (int)cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace));
}
#endif

cudaError_t launch_attention(const AttnProblem &p, cudaStream_t st) {
    if (p.Sq <= 0 || p.n_heads <= 0 || p.B <= 0) return cudaSuccess;
    switch (p.D) {
        case 64: return launch_d<64>(p, st);
        case 96: return launch_d<96>(p, st);
        case 128: return launch_d<128>(p, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace spa
