// attn_fwd.cu -- bf16 flash attention forward for sm_100a on tcgen05 / TMEM / TMA.
//
// Computes, per (batch b, head j, query row s):
//     o[b,s,j,:] = softmax_t( q[b,s,j,:] . k[b,t,j,:] / sqrt(D) ) v[b,t,j,:]
// which is Alg. 1 line 3 `attention(Q[:,j],K[:,j],V[:,j])` for a
// group of heads; the scale 1/sqrt(D) is the north star's (R1).
//
// Design (DESIGN.md §Kernels / attention), one CTA = one 128-row query tile of one (b, head); clusters of
// two CTAs (adjacent query tiles of the same head) share every K/V tile through TMA multicast:
//   warps 0..15  softmax / correction / epilogue: warp w owns TMEM lanes 32*(w%4)..+31 (its rows, = its SM
//                sub-partition) and keys [32*(w/4), 32*(w/4)+32) of every 128-key tile; the 4 warps of a row
//                quarter assemble the row max through shared memory (named barrier) every tile.
//   warp 16      TMA producer: Q once, then K/V tiles through an NS-slot shared-memory ring in the order the
//                MMA consumes them (K0, K1, V0, K2, V1, K3, ...); each CTA fetches 64 of the 128 rows of every
//                tile and multicasts them to both CTAs of the pair.
//   warp 17      TMEM allocator + tcgen05.mma issuer (one elected lane; highest warp id = scheduling priority).
//   TMEM: S double buffer at columns [0,128) and [128,256) (fp32), O at [256, 256+D).
//   * S(j) = Q K_j^T   tcgen05.mma SS, M=128 N=128 into S buffer j%2, so QK^T of tile j+1 runs while the
//     softmax of tile j is in progress.
//   * P(j) (bf16) is written by each softmax warp over the first 16 columns of its own 32 score columns (scores
//     it has already read); key half 0 (keys 0..63) and half 1 are released to the MMA issuer separately.
//   * O += P(j) V_j     tcgen05.mma TS (A = P from TMEM, B = V MN-major, N = D in one instruction).
//   * online softmax in fp32, base 2 with log2(e)/sqrt(D) folded into one FFMA2; the running max only moves
//     when it grows by more than 2^8 (conditional rescale; exact, since the final 1/l uses the same max).  The
//     decision is per row, so a row's result does not depend on the other rows of its tile (bit-identical
//     across stage splits).  A quarter of the exponentials run as a degree-3 polynomial on the FMA pipe.
//   * keys >= Skv (ragged tail, TMA zero-filled) get score -inf; query rows >= Sq are not stored.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "ptx.cuh"
#include "spa_internal.h"

namespace spa {

namespace {

constexpr int BM = 128;        // query rows per CTA (MMA M)
constexpr int BN = 128;        // keys per tile (MMA N of QK^T, K of PV)
// Softmax warps per row quarter: each owns BN/KSPLIT keys of every KV tile for 32 rows.  Four warps
// per SM sub-partition hide the fixed-latency dependency stalls of the exp/sum/pack chain.
constexpr int KSPLIT = 4;
constexpr int KPW = BN / KSPLIT;                 // keys per softmax warp (32)
constexpr int NUM_SOFTMAX_WARPS = 4 * KSPLIT;
constexpr int NUM_WARPS = NUM_SOFTMAX_WARPS + 2;
constexpr int NUM_THREADS = NUM_WARPS * 32;
constexpr int PRODUCER_WARP = NUM_SOFTMAX_WARPS;
// The MMA issuer has the highest warp id: the warp scheduler favours higher ids, and its few instructions
// must not queue behind the softmax warps that share its SM sub-partition.
constexpr int MMA_WARP = NUM_SOFTMAX_WARPS + 1;
constexpr float RESCALE_TAU = 8.0f;  // log2 domain: raise the running max only if it grows by > 2^8

#ifdef SPA_ATTN_TRACE
// Debug timeline of CTA (0,0,0): g_trace[j][e] = clock64 at event e of KV iteration j (tools/attn_trace.py).
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
    static constexpr int NS = (D == 128) ? 5 : 8;         // K/V ring slots
    static constexpr int SMEM_TILES = 1 + NS;
    static constexpr int BAR_BYTES = 256;
    static constexpr int XCH_BYTES = (2 * KSPLIT + KSPLIT) * BM * 4; // static smem: row-max exchange + row sums
    static constexpr int SMEM_BYTES = 1024 /*align slack*/ + SMEM_TILES * TILE_BYTES + BAR_BYTES;
    static constexpr uint32_t TMEM_COLS = 512;           // S0 | S1 | O (power of two >= 256 + D)
    // O columns are handled (rescale, store) in 32-column slices, one per softmax warp kq < D/32, so every
    // tcgen05.ld/st of O is a 32-column-aligned x32 access.
    static constexpr int DW = 32;
    static constexpr int NSLICE = D / 32;
    // exp2 split: key pairs with (i & 7) >= POLY_FROM use the FMA-pipe polynomial, the rest MUFU.EX2.
    // 6 = 1/4 polynomial was fastest at D = 64, 96 and 128 (sweep of 2/4/6/8 on B200).
#ifdef SPA_POLY_FROM
    static constexpr int POLY_FROM = SPA_POLY_FROM;
#else
    static constexpr int POLY_FROM = 6;
#endif
    static_assert(SMEM_BYTES + XCH_BYTES <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ int chunk_off(int c) { return c * (BM * 128); }  // Q/K chunk c byte offset in a tile

struct SmemBars {
    uint64_t q_full;
    uint64_t kv_full[8];
    uint64_t kv_empty[8];
    uint64_t s_full[2];       // [S buffer]
    uint64_t p_full[2][2];    // [S buffer][key half]
    uint64_t o_done;          // one phase per completed PV(j)
    uint64_t o_final;         // all PVs completed (epilogue)
    uint32_t tmem_base;
};

// 2^x on the FMA pipe: x = n + f (n = round(x), |f| <= 1/2), 2^f by a degree-3 fit (max rel err 7.5e-5,
// far below the bf16 rounding of P), 2^n by adding n to the exponent field.  x is clamped at -125 so the
// result stays a normal number (p >= 0.7 has exponent >= 126).

// Two ex2_poly at once in f32x2 arithmetic (same operations per element, so identical results).
__device__ __forceinline__ void ex2_poly2(uint64_t X, float &y0, float &y1) {
    float x0, x1;
    ptx::f2unpack(X, x0, x1);
    const uint64_t Xc = ptx::f2pack(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
    const uint64_t T = ptx::fadd2(Xc, ptx::f2pack(12582912.f, 12582912.f));
    const uint64_t F = ptx::fsub2(Xc, ptx::fadd2(T, ptx::f2pack(-12582912.f, -12582912.f)));
    uint64_t P = ptx::ffma2(ptx::f2pack(0.0551716611f, 0.0551716611f), F, ptx::f2pack(0.242611152f, 0.242611152f));
    P = ptx::ffma2(P, F, ptx::f2pack(0.693260968f, 0.693260968f));
    P = ptx::ffma2(P, F, ptx::f2pack(0.999928057f, 0.999928057f));
    float p0, p1, t0, t1;
    ptx::f2unpack(P, p0, p1);
    ptx::f2unpack(T, t0, t1);
    y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
    y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
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
    uint8_t *sQ = smem;                                        // 1 tile
    uint8_t *sKV = smem + C::TILE_BYTES;                       // NS tiles
    // row-max / row-sum exchange between the KSPLIT warps of a row quarter: a static __shared__ array, so
    // the compiler emits STS/LDS (a pointer derived from the aligned dynamic base would be generic LD/ST)
    __shared__ float xmax[2 * KSPLIT * BM];   // [iteration parity][key slice][row]
    __shared__ float xsum[KSPLIT * BM];       // [key slice][row]
    SmemBars *bars = reinterpret_cast<SmemBars *>(smem + C::SMEM_TILES * C::TILE_BYTES);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int qtile = blockIdx.x;
    const int head = blockIdx.y;
    const int b = blockIdx.z;
    const int n_kv = (args.Skv + BN - 1) / BN;

    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars->q_full, 1);
        for (int i = 0; i < C::NS; ++i) {
            ptx::mbar_init(&bars->kv_full[i], 1);
            ptx::mbar_init(&bars->kv_empty[i], 2);   // released by the MMA issuers of both CTAs of the pair
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&bars->s_full[s], 1);
            // half 0: P written by the warps of keys 0..63 + "O corrected" from the warps of keys 64..127
            // (PV of half 0 updates all of O's columns, so every O slice must be rescaled first)
            ptx::mbar_init(&bars->p_full[s][0], NUM_SOFTMAX_WARPS);
            ptx::mbar_init(&bars->p_full[s][1], NUM_SOFTMAX_WARPS / 2);
        }
        ptx::mbar_init(&bars->o_done, 1);
        ptx::mbar_init(&bars->o_final, 1);
        ptx::fence_mbar_init();
    }
    if (warp == PRODUCER_WARP && lane == 0) {
        ptx::prefetch_tmap(&tmQa); ptx::prefetch_tmap(&tmKa); ptx::prefetch_tmap(&tmVa);
        if (C::N64) { ptx::prefetch_tmap(&tmQb); ptx::prefetch_tmap(&tmKb); ptx::prefetch_tmap(&tmVb); }
    }
    if (warp == MMA_WARP) {
        ptx::tmem_alloc(&bars->tmem_base, C::TMEM_COLS);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();   // the partner's barriers exist before any multicast lands in its shared memory
    ptx::tc_fence_after();
    const uint32_t tmem = bars->tmem_base;
    const uint32_t crank = ptx::cluster_ctarank();   // which half (64 rows) of each K/V tile this CTA fetches

    if (warp == PRODUCER_WARP) {
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
            ptx::mbar_arrive_expect_tx(&bars->q_full, C::TILE_BYTES);
            load_qk(&tmQa, &tmQb, &bars->q_full, sQ, qtile * BM, pol_q);
        }
        int cnt = 0;
        // Each CTA of the pair fetches rows [64*crank, 64*crank+64) of every K/V tile and multicasts them to
        // both CTAs (same smem offset); each CTA's kv_full expects the whole tile.  Halves the L2->SMEM
        // traffic per query row relative to unshared 128-row tiles.
        auto load = [&](bool isV, int j) {
            const int slot = cnt % C::NS;
            ptx::mbar_wait(&bars->kv_empty[slot], ((cnt / C::NS) & 1) ^ 1);
            if (lane == 0) TRACE(j, isV ? 7 : 2);
            if (lane == 0) {
                uint8_t *dst = sKV + slot * C::TILE_BYTES;
                uint64_t *bar = &bars->kv_full[slot];
                ptx::mbar_arrive_expect_tx(bar, C::TILE_BYTES);
                const int row = j * BN + (int)crank * (BN / 2);
                if (isV) {
                    const CUtensorMap *mv = &tmVa;
#pragma unroll
                    for (int a = 0; a < C::V_ATOMS; ++a)
                        ptx::tma_load_4d_mc(mv, bar, dst + a * C::V_ATOM_BYTES + crank * (C::V_ATOM_BYTES / 2),
                                            a * C::V_ATOM_COLS, head, row, b, 0x3, pol_kv);
                } else {
                    ptx::tma_load_4d_mc(&tmKa, bar, dst + crank * (BM / 2) * 128, 0, head, row, b, 0x3, pol_kv);
                    if (C::N128 == 2)
                        ptx::tma_load_4d_mc(&tmKa, bar, dst + chunk_off(1) + crank * (BM / 2) * 128, 64, head, row,
                                            b, 0x3, pol_kv);
                    if (C::N64)
                        ptx::tma_load_4d_mc(&tmKb, bar, dst + chunk_off(1) + crank * (BM / 2) * 64, 64, head, row, b,
                                            0x3, pol_kv);
                }
            }
            __syncwarp();
            ++cnt;
        };
        // same order as the MMA issuer consumes: K0, K1, then V_j, K_{j+2}
        load(false, 0);
        if (n_kv > 1) load(false, 1);
        for (int j = 0; j < n_kv; ++j) {
            load(true, j);
            if (j + 2 < n_kv) load(false, j + 2);
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer
        constexpr uint32_t IDESC_QK = ptx::idesc_bf16(BM, BN, 0, 0);
        constexpr uint32_t IDESC_PV = ptx::idesc_bf16(BM, D, 0, 1);
        const uint32_t qa = ptx::smem_u32(sQ);
        const uint32_t sKV_addr = ptx::smem_u32(sKV);
        const uint32_t tO = tmem + 256;

        int cnt = 0;
        auto acquire = [&]() -> int {   // next ring slot, waiting for its data
            const int slot = cnt % C::NS;
            ptx::mbar_wait(&bars->kv_full[slot], (cnt / C::NS) & 1);
            ptx::tc_fence_after();
            ++cnt;
            return slot;
        };
        // Descriptors are built once; per MMA only the 14-bit start-address field moves (+byte offset >> 4).
        const uint64_t dQ128 = ptx::smem_desc(qa, 16, 1024, 2), dQ64 = ptx::smem_desc(qa + chunk_off(1), 16, 512, 4);
        const uint64_t dK128 = ptx::smem_desc(sKV_addr, 16, 1024, 2);
        const uint64_t dK64 = ptx::smem_desc(sKV_addr + chunk_off(1), 16, 512, 4);
        constexpr uint32_t rowb = C::V_ATOM_COLS * 2;
        const uint64_t dV = ptx::smem_desc(sKV_addr, C::V_ATOM_BYTES, 8 * rowb, C::V_SW64 ? 4u : 2u);
        const bool leader = ptx::elect_one();
        // S(j) = Q K_j^T into S buffer j%2: K-major A (Q) and B (K), 16-element k-steps per swizzle chunk.
        auto issue_qk = [&](int j) {
            if (leader) TRACE(j, 12);
            const int slot = acquire();
            if (leader) {
                TRACE(j, 13);
                const uint64_t so = (uint64_t)(slot * C::TILE_BYTES) >> 4;
                const uint32_t d = tmem + (j & 1) * 128;
#pragma unroll
                for (int c = 0; c < C::NCHUNK; ++c) {
                    const bool sw64 = (c >= C::N128);
                    const int ksteps = sw64 ? 2 : 4;
#pragma unroll
                    for (int kk = 0; kk < ksteps; ++kk) {
                        const uint64_t off = (uint64_t)((sw64 ? 0 : c * (BM * 128)) + kk * 32) >> 4;
                        const uint64_t ad = (sw64 ? dQ64 : dQ128) + off;
                        const uint64_t bd = (sw64 ? dK64 : dK128) + so + off;
                        ptx::mma_ss(d, ad, bd, IDESC_QK, (c | kk) ? 1u : 0u);
                    }
                }
                ptx::mma_commit(&bars->s_full[j & 1]);
                ptx::mma_commit_mc(&bars->kv_empty[slot], 0x3);
            }
            __syncwarp();
        };

        ptx::mbar_wait(&bars->q_full, 0);
        issue_qk(0);
        if (n_kv > 1) issue_qk(1);
        for (int j = 0; j < n_kv; ++j) {
            const int buf = j & 1;
            const uint32_t tS = tmem + buf * 128;
            if (leader) TRACE(j, 14);
            const int slotV = acquire();
            if (leader) TRACE(j, 15);
            const uint64_t dVs = dV + ((uint64_t)(slotV * C::TILE_BYTES) >> 4);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                ptx::mbar_wait(&bars->p_full[buf][hf], (j >> 1) & 1);
                ptx::tc_fence_after();
                if (leader) {
                    TRACE(j, hf);
                    // O (+)= P(j)[keys 64hf..64hf+63] V_j[those keys]; the P of keys [KPW*k, KPW*k+KPW) sits in
                    // columns [KPW*k, KPW*k + KPW/2) (written over scores its warp had already read)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const int key16 = hf * 4 + kk;
                        const int pcol = (key16 * 16 / KPW) * KPW + (key16 * 16 % KPW) / 2;
                        ptx::mma_ts(tO, tS + pcol, dVs + ((uint64_t)(key16 * 16 * rowb) >> 4), IDESC_PV,
                                    (j > 0 || key16 > 0) ? 1u : 0u);
                    }
                    if (hf == 1) {
                        ptx::mma_commit(&bars->o_done);
                        if (j == n_kv - 1) ptx::mma_commit(&bars->o_final);
                        ptx::mma_commit_mc(&bars->kv_empty[slotV], 0x3);
                    }
                }
                __syncwarp();
            }
            if (j + 2 < n_kv) issue_qk(j + 2);
        }
    } else {
        // ------------------------------------------------------------ softmax / correction / epilogue
        const int kq = warp >> 2;                      // key slice [KPW*kq, KPW*kq + KPW) of every KV tile
        const int wq = warp & 3;                       // TMEM lane quarter this warp may access (= SMSP)
        const int row = wq * 32 + lane;                // row within the tile
        const int hf = kq / (KSPLIT / 2);              // which P half (keys 0..63 / 64..127) this warp feeds
        const uint32_t bar_id = 1 + wq;                // named barrier of the KSPLIT warps sharing these rows
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        const uint32_t tO = tmem + lane_base + 256 + kq * C::DW;   // this warp's slice of O's columns
        const float sl2 = args.scale_log2;
        const int last_valid = args.Skv - (n_kv - 1) * BN;   // valid keys in the last tile (1..128)
        const int key0 = kq * KPW;
        const bool tr = (lane == 0 && wq == 0 && (kq % (KSPLIT / 2)) == 0);

        float m = -INFINITY;   // running max, already scaled to the log2 domain (same in all KSPLIT warps)
        float l = 0.f;         // this warp's running sum of p (fp32)
        for (int j = 0; j < n_kv; ++j) {
            const int buf = j & 1;
            const uint32_t tS = tmem + lane_base + buf * 128 + key0;   // this warp's KPW scores
            const bool masked = (j == n_kv - 1) && (last_valid < BN);
            if (tr) TRACE(j, 3 + 5 * hf);
            ptx::mbar_wait(&bars->s_full[buf], (j >> 1) & 1);
            ptx::tc_fence_after();
            if (tr) TRACE(j, 4 + 5 * hf);
            // One TMEM read of this warp's KPW scores: slice max -> row max assembled from the KSPLIT slices
            // through shared memory -> conditional rescale -> P.
            uint32_t sv[KPW];
            ptx::tmem_ld_cols<KPW>(tS, sv);
            ptx::tmem_wait_ld();
            if (masked) {
#pragma unroll
                for (int i = 0; i < KPW; ++i)
                    if (key0 + i >= last_valid) sv[i] = __float_as_uint(-INFINITY);
            }
            uint32_t pk[KPW / 2];
            float lsum;
            auto exps = [&](float mcur) {
                const uint64_t SL2 = ptx::f2pack(sl2, sl2), NEGM = ptx::f2pack(-mcur, -mcur);
                uint64_t L0 = ptx::f2pack(0.f, 0.f), L1 = L0;
#pragma unroll
                for (int i = 0; i < KPW / 2; ++i) {
                    const uint64_t X = ptx::ffma2(ptx::f2pack(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])),
                                                  SL2, NEGM);
                    float p0, p1;
                    if (((2 * i) & 7) >= C::POLY_FROM) {
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
                float a0, a1, b0, b1;
                ptx::f2unpack(L0, a0, a1);
                ptx::f2unpack(L1, b0, b1);
                lsum = (a0 + b0) + (a1 + b1);
            };
            float mx;
            {
                float m0 = __uint_as_float(sv[0]), m1 = __uint_as_float(sv[1]);
#pragma unroll
                for (int i = 2; i < KPW; i += 2) {
                    m0 = fmaxf(m0, __uint_as_float(sv[i]));
                    m1 = fmaxf(m1, __uint_as_float(sv[i + 1]));
                }
                mx = fmaxf(m0, m1);
            }
            float *xm = xmax + (j & 1) * KSPLIT * BM;
            xm[kq * BM + row] = mx;
            ptx::named_bar_sync(bar_id, 32 * KSPLIT);
#pragma unroll
            for (int k = 0; k < KSPLIT; ++k) mx = fmaxf(mx, xm[k * BM + row]);
            mx *= sl2;
            if (tr) TRACE(j, 5 + 5 * hf);
            const bool resc = mx > m + RESCALE_TAU;      // also true on the first tile (m = -inf)
            if (__any_sync(0xffffffffu, resc)) {
                float factor = 1.f;
                if (resc) {
                    factor = ptx::ex2(m - mx);            // 0 on the first tile
                    m = mx;
                }
                l *= factor;
                // O *= factor for the moved rows (others by exactly 1) after PV(j-1) completed and before
                // PV(j) of either key half (the half-0 PV also updates this warp's O slice).
                if (j > 0 && kq < C::NSLICE) {
                    // unambiguous: S(j) completed, so PV(j-2) did (issued before QK(j)); o_done is <= 1 phase behind
                ptx::mbar_wait(&bars->o_done, (j - 1) & 1);
                    ptx::tc_fence_after();
                    uint32_t r[C::DW];
                    ptx::tmem_ld_cols<C::DW>(tO, r);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < C::DW; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * factor);
                    ptx::tmem_st_cols<C::DW>(tO, r);
                    ptx::tmem_wait_st();
                }
            }
            exps(m);
            l += lsum;
            if (hf == 1) {   // this warp's O slice is ready for PV(j) of key half 0
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&bars->p_full[buf][0]);
            }
            ptx::tmem_st_cols<KPW / 2>(tS, pk);   // over scores this warp has already consumed
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&bars->p_full[buf][hf]);
            if (tr) TRACE(j, 6 + 5 * hf);
        }
        // ------------------------------------------------------------ epilogue: O / l -> bf16 -> global
        xsum[kq * BM + row] = l;
        ptx::named_bar_sync(bar_id, 32 * KSPLIT);
        float lsum = 0.f;
#pragma unroll
        for (int k = 0; k < KSPLIT; ++k) lsum += xsum[k * BM + row];
        const float inv_l = 1.f / lsum;
        ptx::mbar_wait(&bars->o_final, 0);   // (o_done could be two phases behind here)
        ptx::tc_fence_after();
        const long long srow = (long long)qtile * BM + row;
        const bool valid = srow < args.Sq;      // tcgen05.ld is warp-collective: every lane loads, valid lanes store
        if (kq < C::NSLICE) {   // warps kq >= D/32 own no O slice (D = 64 / 96)
            uint32_t r[C::DW];
            ptx::tmem_ld_cols<C::DW>(tO, r);
            ptx::tmem_wait_ld();
            if (valid) {
                uint4 *dst = reinterpret_cast<uint4 *>(args.O + (long long)b * args.o_batch_stride +
                                                       srow * args.o_tok_stride + (long long)head * D + kq * C::DW);
#pragma unroll
                for (int v = 0; v < C::DW / 8; ++v) {
                    uint32_t w[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        w[u] = ptx::pack_bf16x2(__uint_as_float(r[8 * v + 2 * u]) * inv_l,
                                                __uint_as_float(r[8 * v + 2 * u + 1]) * inv_l);
                    dst[v] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();   // no CTA leaves while its partner may still multicast into it / arrive on its barriers
    if (warp == MMA_WARP) {
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

// 4-D map over a [B][S][heads][D] bf16 view: dims (D, heads, S, B), box (box_d, 1, box_rows, 1).
bool make_map(CUtensorMap *m, const void *base, int D, int heads, int S, int B, long long tok_stride,
              long long batch_stride, int box_d, bool sw64, int box_rows = BM) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)heads, (cuuint64_t)S, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)tok_stride * 2, (cuuint64_t)batch_stride * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_d, 1, (cuuint32_t)box_rows, 1};
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
    // m[0]/m[1]: Q 64-col SW128 / 32-col SW64 boxes of 128 rows; m[2]/m[3]: the same for K with 64-row boxes
    // (each CTA of a pair fetches half a tile); m[4]: V 64-col SW128 (D=64/128) or 32-col SW64 (D=96) boxes
    // of 64 rows; m[5] unused.
    CUtensorMap m[6];
    const int vcols = C::V_SW64 ? 32 : 64;
    bool ok = make_map(&m[0], p.q, D, p.n_heads, p.Sq, p.B, p.q_tok_stride, p.q_batch_stride, 64, false) &&
              make_map(&m[2], p.k, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, 64, false, BM / 2) &&
              make_map(&m[4], p.v, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, vcols, C::V_SW64,
                       BM / 2);
    if (ok && C::N64)
        ok = make_map(&m[1], p.q, D, p.n_heads, p.Sq, p.B, p.q_tok_stride, p.q_batch_stride, 32, true) &&
             make_map(&m[3], p.k, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, 32, true, BM / 2);
    else {
        m[1] = m[0];
        m[3] = m[2];
    }
    m[5] = m[4];
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
    // clusters of 2 CTAs (adjacent query tiles of one head) share every K/V tile via TMA multicast;
    // an odd tile count gets one extra all-out-of-range tile that only helps its partner load.
    const int qtiles = (p.Sq + BM - 1) / BM;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((qtiles + 1) & ~1, p.n_heads, p.B);
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, attn_fwd_kernel<D>, m[0], m[1], m[2], m[3], m[4], m[5], a);
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
