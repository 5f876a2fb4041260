// attn_fwd.cu -- bf16 flash attention forward for sm_100a on tcgen05 / TMEM / TMA.
//
// Computes, per (batch b, head j, query row s):
//     o[b,s,j,:] = softmax_t( q[b,s,j,:] . k[b,t,j,:] / sqrt(D) ) v[b,t,j,:]
// which is Alg. 1 line 3 `attention(Q[:,j],K[:,j],V[:,j])` for a
// group of heads; the scale 1/sqrt(D) is the north star's (R1).
//
// Design, one CTA = one 128-row query tile of one (b, head); the two CTAs of a cluster
// (adjacent query tiles of the same head) form a CTA PAIR that runs every MMA as one tcgen05 cta_group::2
// instruction (M = 256): each CTA holds its own Q tile and only HALF of every K tile (64 keys) and V tile
// (D/2 columns), so each SM takes in half of the K/V stream; only the leader CTA issues MMAs.
//   * TMEM: three S buffers (fp32, 128 columns each) at [0,128), [128,256), [256,384) and ONE O
//     accumulator at [384, 384+D).  KV tile j goes to S buffer j%3 and is handled by softmax group j%3
//     (group g = warps 4+4g..7+4g, one warp per TMEM lane quarter = SM sub-partition).  Three S buffers make
//     three independent S -> softmax -> PV chains, so the tensor pipe always has a QK^T or PV product
//     queued while a group is in its softmax (each group has three tiles of MMA time for one tile of
//     softmax; the v3 design with two chains was latency-bound: softmax warps idled a third of the time
//     on S(j)).
//   * The running max is one per row, shared by all groups: it travels tile to tile through shared
//     memory (named barrier arrive/sync between the warps of consecutive groups on the same sub-partition),
//     so every P is relative to the same reference max as O.  It only moves when a tile's row max exceeds
//     it by more than 2^8 (conditional rescale); then the group that moved it waits for PV(j-1) and rescales
//     O in TMEM before releasing P(j).  Each group keeps its own partial row sum l_g relative to the last
//     max it saw; the epilogue merges them.
//   warp 0 TMA producer (warps 1, 2 idle): Q once, then K/V tiles through an NS-slot smem ring in consumption order
//           (K0, K1, K2, V0, K3, V1, K4, ...); each CTA of the pair loads only its half of every tile (64 keys
//           of K, D/2 columns of V), counted on the leader's full barrier.
//   warp 3 TMEM allocator (cta_group::2, both CTAs) + tcgen05.mma issuer (leader CTA, one elected lane; the
//           softmax warps 4.. have the higher ids = scheduler priority): S(j) = Q K_j^T (SS, M=256, N=128) into S buffer j%3 of both CTAs;
//           O += P(j) V_j (TS: P from each CTA's TMEM, V MN-major, N = D in one instruction), released in two
//           key halves once the softmax warps of BOTH CTAs arrived (8 arrivals on the leader's barrier);
//           S(j+3) is issued right after PV(j).  Commits are multicast to both CTAs' barriers.
//   * softmax (one thread per row, 128 keys): two-pass over TMEM (row max, then exp2 in two 64-key halves,
//     each released to the MMA issuer as soon as its bf16 P is in TMEM, written over scores already read);
//     fp32, base 2 with log2(e)/sqrt(D) folded into one FFMA2; a quarter of the exponentials run as a
//     degree-3 polynomial on the FMA pipe.  Every decision is per row and the group of a tile depends only
//     on its index, so a row's result does not depend on which other rows share its tile (bit-identical
//     across stage splits).
//   * keys >= Skv (ragged tail, TMA zero-filled) get score -inf; query rows >= Sq are not stored.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>

#include "ptx.cuh"
#include "spa_internal.h"

namespace spa {

namespace {

constexpr int BM = 128;        // query rows per CTA (MMA M)
constexpr int NG_MAX = 4;
constexpr float RESCALE_TAU = 8.0f;   // log2 domain: raise the running max only if it grows by > 2^8
// CTA pair: clusters of 2 adjacent query tiles of one head run every MMA as ONE cta_group::2 instruction
// (M = 256); each CTA holds only half of every K tile (64 keys) and half of every V tile (D/2 columns), so
// each SM takes in half of the K/V stream (the L2->SMEM feed was the first limiter of the M = 128 design).
constexpr uint16_t PAIR_MASK = 0x3;
// Order in which the softmax releases (and the MMA consumes) the two 64-key halves of P: the upper half first,
// straight from the registers pass 1 loaded last (one TMEM read of 64 columns per tile saved).
__device__ constexpr int HALF_ORDER[2] = {1, 0};



#ifdef SPA_ATTN_TRACE
// Debug timeline of CTA (0,0,0): g_trace[j][e] = clock64 at event e of KV iteration j (tools/attn_trace.py).
__device__ unsigned long long g_trace[256][16];
#define TRACE(j, e)                                                                  \
    do {                                                                             \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 256)      \
            g_trace[(j)][(e)] = clock64();                                           \
    } while (0)
// per softmax warp of both CTAs of cluster 0: [j][crank*4 + wq][0] = S(j) seen, [1] = first P half released,
// [2] = second P half released (clock64 of that SM)
__device__ unsigned long long g_trace2[256][8][3];
#define TRACE2(j, slot, e)                                                                     \
    do {                                                                                      \
        if (blockIdx.x < 2 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 256 && lane == 0)    \
            g_trace2[(j)][(slot)][(e)] = clock64();                                           \
    } while (0)
#else
#define TRACE(j, e) do {} while (0)
#define TRACE2(j, slot, e) do {} while (0)
#endif

template <int D>
struct Cfg {
    static_assert(D == 64 || D == 96 || D == 128, "D in {64, 96, 128}");
    // Keys per KV tile (MMA N of QK^T, K of PV) and softmax groups = S buffers in TMEM = independent
    // S -> softmax -> PV chains: three chains of 128-key tiles.  SPA_NG4_D96 builds D=96 with four chains of
    // 96-key tiles (4 x 96 + 96 = 480 TMEM columns, 104 softmax registers); measured 1-3 % slower
    // (profiles/r01_v5_experiments/README.md), so it is not the default.
#ifndef SPA_NG4_MASK
#ifdef SPA_NG4_D96
#define SPA_NG4_MASK 2
#else
#define SPA_NG4_MASK 0   // bit 0: D = 64, bit 1: D = 96, bit 2: D = 128 -> four chains of 96-key tiles
#endif
#endif
    static constexpr bool NG4 = ((SPA_NG4_MASK >> (D == 64 ? 0 : (D == 96 ? 1 : 2))) & 1) != 0;
    // DP: "decoupled P" -- three chains of 96-key tiles whose bf16 P goes to two separate TMEM P buffers instead of over
    // the scores, so a tile's S buffer is free as soon as pass 1 has read it (both halves stay in registers) and S(j+3)
    // is issued then, not after PV(j): the MMA chain no longer waits for the softmax's exponentials.
#ifndef SPA_DP_MASK
#define SPA_DP_MASK 0   // bit 0: D = 64, bit 1: D = 96, bit 2: D = 128
#endif
    static constexpr bool DP = !NG4 && ((SPA_DP_MASK >> (D == 64 ? 0 : (D == 96 ? 1 : 2))) & 1) != 0;
    static constexpr int BN = (NG4 || DP) ? 96 : 128;
    static constexpr int NG = NG4 ? 4 : 3;
    static constexpr int HALF = BN / 2;                  // keys per P release (64 or 48)
    static constexpr int NUM_SOFTMAX_WARPS = 4 * NG;
    // Warpgroup 0 = {producer, 2 idle, MMA issuer}, then NG warpgroups of softmax warps.  Warpgroup 0 gives its
    // registers to the softmax warps (setmaxnreg): per SM sub-partition NG x SOFTMAX_REGS + AUX_REGS <=
    // (NG + 1) x LAUNCH_REGS.  The softmax warps have the higher warp ids, i.e. the scheduler's priority over the
    // producer and MMA warps that share SM sub-partitions 0 and 3 with them (measured +0.2..1.4 % over the
    // opposite order; the per-warp trace shows those two lane quarters are the slowest).
    static constexpr int AUX_BASE = 0, SM_BASE = 4;
    static constexpr int PRODUCER_WARP = AUX_BASE;
    static constexpr int MMA_WARP = AUX_BASE + 3;
    static constexpr int NUM_THREADS = (NUM_SOFTMAX_WARPS + 4) * 32;
    // setmaxnreg only moves registers within the CTA's launch allocation (65536 / NUM_THREADS rounded down to
    // a multiple of 8 per thread: 128 for 512 threads, 96 for 640), so the split must fit that pool.
    static constexpr int LAUNCH_REGS = (65536 / NUM_THREADS) / 8 * 8;
    static constexpr int SOFTMAX_REGS = (NG == 4) ? 104 : 152, AUX_REGS = (NG == 4) ? 64 : 56;
    static_assert(NG * SOFTMAX_REGS + AUX_REGS <= (NG + 1) * LAUNCH_REGS, "register split exceeds the CTA pool");
    // Named barriers (0 = __syncthreads).  NG = 3: 1 + 3*wq + g = "running max of the previous tile is in xm[]
    // for the warp of group g on lane quarter wq" (64 threads); NG = 4 (16 would not fit): 1 + g for the four
    // warps of group g and of the group before it (256 threads).  BAR_EPI: all softmax warps (epilogue merge).
    static constexpr uint32_t BAR_EPI = (NG == 3) ? 13 : 5;
    // Q/K tiles (K-major operands): 64-column 128B-swizzled chunks + (D=96) one 32-column 64B-swizzled chunk.
    static constexpr int N128 = D / 64;                  // 1, 1, 2
    static constexpr int N64 = (D % 64) ? 1 : 0;         // 0, 1, 0
    static constexpr int NCHUNK = N128 + N64;
    // This CTA's half of a V tile (MN-major B operand of PV; the pair's N = D is split D/2 per CTA), as
    // [128 keys][D/2] in swizzle atoms along N: D=128 -> one 64-column SW128 atom, D=64 -> one 32-column SW64
    // atom, D=96 -> three 16-column SW32 atoms; LBO = distance between atoms along N.
    static constexpr int VH = D / 2;
    static constexpr int V_ATOM_COLS = (D == 128) ? 64 : (D == 64 ? 32 : 16);
    static constexpr uint32_t V_LAYOUT = (D == 128) ? 2u : (D == 64 ? 4u : 6u);   // SW128 / SW64 / SW32
    static constexpr int V_ATOMS = VH / V_ATOM_COLS;
    static constexpr int V_ATOM_BYTES = BN * V_ATOM_COLS * 2;
    static constexpr int TILE_BYTES = BM * D * 2;        // Q tile
    static constexpr int KV_TILE_BYTES = BN * D * 2;     // a whole K or V tile of the pair
    static constexpr int HALF_BYTES = KV_TILE_BYTES / 2; // one ring slot: this CTA's half of a K or V tile
    static constexpr int KCHUNK = (BN / 2) * 128;        // K half: BN/2 keys; 64-column SW128 chunk c at c*KCHUNK
    // K/V ring slots (as many as fit: the ring depth is the TMA lookahead that hides L2 latency)
    static constexpr int NS = (D == 128 && BN == 128) ? 12 : 16;
    static constexpr int BAR_BYTES = 512;
    static constexpr int XCH_BYTES = BM * 4;   // static smem: running max (the epilogue's (m, l) reuse ring slot 0)
    static constexpr int SMEM_BYTES = 1024 /*align slack*/ + TILE_BYTES + NS * HALF_BYTES + BAR_BYTES;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr uint32_t P_COL = BN * NG;           // DP: P buffers u = 0, 1 at [P_COL + u*HALF, +HALF)
    static constexpr uint32_t O_COL = BN * NG + (DP ? BN : 0);   // O accumulator columns [O_COL, O_COL + D)
    static_assert(O_COL + D <= TMEM_COLS, "TMEM budget");
    static constexpr int OCHUNKS = D / 16;               // epilogue: 16-column chunks, chunk c by group c % NG
    // exp2 split: key pairs with (key & 15) >= POLY_FROM use the FMA-pipe polynomial, the rest MUFU.EX2
    // (POLY_FROM = 12: a quarter of the keys on the FMA pipe; 14: an eighth; 16: none).
#ifdef SPA_POLY_FROM
    static constexpr int POLY_FROM = SPA_POLY_FROM;
#else
    // 1/4 on the FMA pipe at every D: interleaved in-process A/B (tools/ab.py, profiles/r02/softmax_ceiling/): at D=96
    // 1/4 beats 1/8 by 1.4-2.5 % (three boxes), 3/8 is equal, 1/2 worse; at D=64 3/8 and 1/8 are 1-2 % slower
    static constexpr int POLY_FROM = 12;
#endif
    static_assert(SMEM_BYTES + XCH_BYTES <= 227 * 1024, "shared memory");
    static_assert(NS <= 16, "barrier block");
    static_assert(2 * NG * BM * 4 <= HALF_BYTES, "epilogue exchange fits in a ring slot");
};

__device__ __forceinline__ int chunk_off(int c) { return c * (BM * 128); }  // Q/K chunk c byte offset in a tile

struct SmemBars {
    uint64_t q_full;
    uint64_t kv_full[16];      // leader's count the data of both CTAs' halves (follower's unused)
    uint64_t kv_empty[16];
    uint64_t s_full[NG_MAX];       // [buffer]: S(j) complete
    uint64_t p_full[NG_MAX][2];    // [buffer][key half]: P(j) half written (leader's: 4 warps of the group, both CTAs)
    uint64_t pv_done[NG_MAX];      // [buffer]: PV(j) complete (O may be rescaled); DP: [j % 4]
    uint64_t s_free[NG_MAX];       // DP: [buffer]: S(j) read by the 8 softmax warps of the pair (S(j+NG) may overwrite it)
    uint64_t o_final;          // all PVs completed (epilogue)
    uint32_t tmem_base;
};
static_assert(sizeof(SmemBars) <= 512, "barrier block");

// Two exp2 at once in f32x2 arithmetic: x = n + f (n = round(x), |f| <= 1/2), 2^f by a degree-3 fit (max rel
// err 7.5e-5, far below the bf16 rounding of P), times 2^n built in the exponent field.  x is clamped to -127,
// where the scale's exponent field is 0: 2^x < 2^-126.5 (and a masked key's -inf) gives exactly 0, like the
// flush-to-zero MUFU.EX2 path.
__device__ __forceinline__ void ex2_poly2(uint64_t X, float &y0, float &y1) {
    float x0, x1;
    ptx::f2unpack(X, x0, x1);
    const uint64_t Xc = ptx::f2pack(fmaxf(x0, -127.f), fmaxf(x1, -127.f));
    const uint64_t T = ptx::fadd2(Xc, ptx::f2pack(12582912.f, 12582912.f));   // 1.5*2^23: low bits = round(x)
    const uint64_t F = ptx::fsub2(Xc, ptx::fadd2(T, ptx::f2pack(-12582912.f, -12582912.f)));
    uint64_t P = ptx::ffma2(ptx::f2pack(0.0551716611f, 0.0551716611f), F, ptx::f2pack(0.242611152f, 0.242611152f));
    P = ptx::ffma2(P, F, ptx::f2pack(0.693260968f, 0.693260968f));
    P = ptx::ffma2(P, F, ptx::f2pack(0.999928057f, 0.999928057f));
    float t0, t1;
    ptx::f2unpack(T, t0, t1);
    // bits(T) = bits(1.5*2^23) + n and bits(1.5*2^23) << 23 == 0 (mod 2^32): one IMAD gives bits(2^n) = (n+127) << 23
    const float s0 = __int_as_float(__float_as_int(t0) * (1 << 23) + (127 << 23));
    const float s1 = __int_as_float(__float_as_int(t1) * (1 << 23) + (127 << 23));
    ptx::f2unpack(ptx::fmul2(P, ptx::f2pack(s0, s1)), y0, y1);
}

template <int D>
__global__ void __launch_bounds__(Cfg<D>::NUM_THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQa, const __grid_constant__ CUtensorMap tmQb,
                    const __grid_constant__ CUtensorMap tmKa, const __grid_constant__ CUtensorMap tmKb,
                    const __grid_constant__ CUtensorMap tmVa, const __grid_constant__ CUtensorMap tmVb,
                    const AttnArgs args) {
    using C = Cfg<D>;
    constexpr int BN = C::BN, NG = C::NG, HALF = C::HALF;
    constexpr int NUM_SOFTMAX_WARPS = C::NUM_SOFTMAX_WARPS, PRODUCER_WARP = C::PRODUCER_WARP, MMA_WARP = C::MMA_WARP;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sQ = smem;                                        // this CTA's Q tile
    uint8_t *sKV = smem + C::TILE_BYTES;                       // NS half tiles
    SmemBars *bars = reinterpret_cast<SmemBars *>(smem + C::TILE_BYTES + C::NS * C::HALF_BYTES);
    __shared__ float xm[BM];            // running max handed from the group of tile j-1 to the group of tile j
    // epilogue: xml[g] = last max seen by group g, xml[NG + g] = its partial sum; in ring slot 0, which is idle once
    // every MMA of this CTA completed (o_final): all loads into this CTA's ring were consumed by then.
    float (*xml)[BM] = reinterpret_cast<float (*)[BM]>(sKV);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int qtile = blockIdx.x;
    const int head = blockIdx.y;
    const int b = blockIdx.z;
    // key-padding mask (Alg. 1 attention_mask; R20): keys t >= kv_len[b] take no
    // part; tiles wholly beyond it are never loaded.  Both CTAs of a cluster share b, hence n_kv.
    int Skv_b = args.Skv;
    if (args.kv_len) {   // key t of this launch is global key t + kv_offset (ring blocks)
        const int L = __ldg(args.kv_len + b) - args.kv_offset;
        Skv_b = L < 0 ? 0 : (L < Skv_b ? L : Skv_b);
    }
    const int n_kv = (Skv_b + BN - 1) / BN;   // 0: every row of this batch entry is 0

    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars->q_full, 1);
        for (int i = 0; i < C::NS; ++i) {
            ptx::mbar_init(&bars->kv_full[i], 1);
            ptx::mbar_init(&bars->kv_empty[i], 1);   // the leader's commit, multicast to both CTAs
        }
        for (int t = 0; t < NG; ++t) {
            ptx::mbar_init(&bars->s_full[t], 1);
            ptx::mbar_init(&bars->p_full[t][0], 8);   // one arrival per softmax warp of that group, both CTAs
            ptx::mbar_init(&bars->p_full[t][1], 8);
            ptx::mbar_init(&bars->pv_done[t], 1);
            if (C::DP) ptx::mbar_init(&bars->s_free[t], 8);   // one arrival per softmax warp of the pair
        }
        if (C::DP) ptx::mbar_init(&bars->pv_done[3], 1);   // DP: PV(j) completes on pv_done[j % 4]
        ptx::mbar_init(&bars->o_final, 1);
        ptx::fence_mbar_init();
    }
    if (warp == PRODUCER_WARP && lane == 0) {
        ptx::prefetch_tmap(&tmQa); ptx::prefetch_tmap(&tmKa); ptx::prefetch_tmap(&tmVa);
        if (C::N64) { ptx::prefetch_tmap(&tmQb); ptx::prefetch_tmap(&tmKb); }
    }
    if (warp == MMA_WARP) {   // same warp id in both CTAs (cta_group::2 allocation)
        ptx::tmem_alloc2(&bars->tmem_base, C::TMEM_COLS);
        ptx::tmem_relinquish2();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();   // the peer's barriers exist before any TMA / commit / arrive targets them
    ptx::tc_fence_after();
    const uint32_t tmem = bars->tmem_base;
    const uint32_t crank = ptx::cluster_ctarank();   // 0 = leader (issues the pair's MMAs)

    if (warp == PRODUCER_WARP) {
        // ------------------------------------------------------------ TMA producer
        ptx::setmaxnreg_dec<C::AUX_REGS>();
        const uint64_t pol_q = ptx::policy_evict_first();
        const uint64_t pol_kv = ptx::policy_evict_last();
        // Every load of either CTA is counted on the LEADER's barrier, which expects the pair's bytes.
        if (lane == 0 && n_kv > 0) {
            const uint32_t qbar = ptx::mapa(&bars->q_full, 0);
            if (crank == 0) ptx::mbar_arrive_expect_tx(&bars->q_full, 2 * C::TILE_BYTES);
            ptx::tma_load_4d_2sm(&tmQa, qbar, sQ, 0, head, qtile * BM, b, pol_q);
            if (C::N128 == 2) ptx::tma_load_4d_2sm(&tmQa, qbar, sQ + chunk_off(1), 64, head, qtile * BM, b, pol_q);
            if (C::N64) ptx::tma_load_4d_2sm(&tmQb, qbar, sQ + chunk_off(1), 64, head, qtile * BM, b, pol_q);
        }
        int cnt = 0;
        // K half: keys [j*BN + crank*BN/2, +BN/2) of tile j, all D columns; V half: all BN keys, columns
        // [crank*D/2, +D/2).  A slot is refilled once the pair's MMA that read it completed (kv_empty).
        auto load = [&](bool isV, int j) {
            const int slot = cnt % C::NS;
            ptx::mbar_wait(&bars->kv_empty[slot], ((cnt / C::NS) & 1) ^ 1);
            if (lane == 0) {
                uint8_t *dst = sKV + slot * C::HALF_BYTES;
                const uint32_t bar = ptx::mapa(&bars->kv_full[slot], 0);
                if (crank == 0) ptx::mbar_arrive_expect_tx(&bars->kv_full[slot], C::KV_TILE_BYTES);
                auto tl = [&](const CUtensorMap *m, uint8_t *d, int c0, int row) {
                    ptx::tma_load_4d_2sm(m, bar, d, c0, head, row, b, pol_kv);
                };
                TRACE(j, isV ? 12 : 11);
                if (isV) {
#pragma unroll
                    for (int a = 0; a < C::V_ATOMS; ++a)
                        tl(&tmVa, dst + a * C::V_ATOM_BYTES, (int)crank * C::VH + a * C::V_ATOM_COLS, j * BN);
                } else {
                    const int row = j * BN + (int)crank * (BN / 2);
                    tl(&tmKa, dst, 0, row);
                    if (C::N128 == 2) tl(&tmKa, dst + C::KCHUNK, 64, row);
                    if (C::N64) tl(&tmKb, dst + C::KCHUNK, 64, row);
                }
            }
            __syncwarp();
            ++cnt;
        };
        // same order as the MMA issuer consumes: K0 .. K_{NG-1}, then V_j, K_{j+NG} (DP: K_{j+NG}, V_j)
        for (int j = 0; j < NG && j < n_kv; ++j) load(false, j);
        for (int j = 0; j < n_kv; ++j) {
            if (C::DP && j + NG < n_kv) load(false, j + NG);
            load(true, j);
            if (!C::DP && j + NG < n_kv) load(false, j + NG);
        }
    } else if (warp == MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer
        ptx::setmaxnreg_dec<C::AUX_REGS>();
        constexpr uint32_t IDESC_QK = ptx::idesc_bf16(2 * BM, BN, 0, 0);   // the pair: M = 256
        constexpr uint32_t IDESC_PV = ptx::idesc_bf16(2 * BM, D, 0, 1);
        const uint32_t qa = ptx::smem_u32(sQ);
        const uint32_t sKV_addr = ptx::smem_u32(sKV);

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
        const uint64_t dK64 = ptx::smem_desc(sKV_addr + C::KCHUNK, 16, 512, 4);
        constexpr uint32_t rowb = C::V_ATOM_COLS * 2;
        const uint64_t dV = ptx::smem_desc(sKV_addr, C::V_ATOM_BYTES, 8 * rowb, C::V_LAYOUT);
        // only the leader CTA issues (one elected lane); the follower's MMA warp just owns its TMEM allocation
        const bool leader = (crank == 0) && ptx::elect_one();
        const uint32_t tO = tmem + C::O_COL;
        // S(j) = Q K_j^T into S buffer j%NG: K-major A (Q) and B (K), 16-element k-steps per swizzle chunk.
        auto issue_qk = [&](int j) {
            const int slot = acquire();
            if (leader) {
                TRACE(j, 2);
                const uint64_t so = (uint64_t)(slot * C::HALF_BYTES) >> 4;
                const uint32_t d = tmem + (j % NG) * BN;
#pragma unroll
                for (int c = 0; c < C::NCHUNK; ++c) {
                    const bool sw64 = (c >= C::N128);
                    const int ksteps = sw64 ? 2 : 4;
#pragma unroll
                    for (int kk = 0; kk < ksteps; ++kk) {
                        const uint64_t qoff = (uint64_t)((sw64 ? 0 : c * (BM * 128)) + kk * 32) >> 4;
                        const uint64_t koff = (uint64_t)((sw64 ? 0 : c * C::KCHUNK) + kk * 32) >> 4;
                        ptx::mma_ss2(d, (sw64 ? dQ64 : dQ128) + qoff, (sw64 ? dK64 : dK128) + so + koff, IDESC_QK,
                                     (c | kk) ? 1u : 0u);
                    }
                }
                ptx::mma_commit2_mc(&bars->s_full[j % NG], PAIR_MASK);
                ptx::mma_commit2_mc(&bars->kv_empty[slot], PAIR_MASK);
            }
            __syncwarp();
        };

        if (crank == 0) {
            if (n_kv > 0) ptx::mbar_wait(&bars->q_full, 0);
            for (int j = 0; j < NG && j < n_kv; ++j) issue_qk(j);
            for (int j = 0; j < n_kv; ++j) {
                const int t = j % NG;
                const uint32_t tS = tmem + t * BN;
                if (C::DP && j + NG < n_kv) {   // S buffer t is free once the 8 softmax warps of tile j read it
                    ptx::mbar_wait(&bars->s_free[t], (j / NG) & 1);
                    ptx::tc_fence_after();
                    issue_qk(j + NG);
                }
                // P(j): over the first HALF/2 columns of each half of S buffer t, or (DP) in P buffer j % 2
                const uint32_t tPj = C::DP ? tmem + C::P_COL + (j & 1) * HALF : tS;
                const int slotV = acquire();
                if (leader) TRACE(j, 10);
                const uint64_t dVs = dV + ((uint64_t)(slotV * C::HALF_BYTES) >> 4);
#pragma unroll
                for (int o = 0; o < 2; ++o) {
                    const int hf = HALF_ORDER[o];   // the key half the softmax releases o-th
                    if (C::DP) ptx::mbar_wait(&bars->p_full[j & 1][hf], (j >> 1) & 1);
                    else ptx::mbar_wait(&bars->p_full[t][hf], (j / NG) & 1);   // both CTAs' softmax warps
                    ptx::tc_fence_after();
                    if (leader) {
                        TRACE(j, o);
                        // O (+)= P(j)[keys HALF*hf ..+HALF) V_j[those keys]; that P half (bf16 pairs) sits in columns
                        // HALF*hf .. HALF*hf + HALF/2 of the S buffer
#pragma unroll
                        for (int kk = 0; kk < HALF / 16; ++kk) {
                            const int key16 = hf * (HALF / 16) + kk;
                            ptx::mma_ts2(tO, tPj + hf * (C::DP ? HALF / 2 : HALF) + kk * 8,
                                         dVs + ((uint64_t)(key16 * 16 * rowb) >> 4),
                                         IDESC_PV, (j > 0 || o > 0 || kk > 0) ? 1u : 0u);
                        }
                        if (o == 1) {
                            ptx::mma_commit2_mc(&bars->kv_empty[slotV], PAIR_MASK);
                            ptx::mma_commit2_mc(&bars->pv_done[C::DP ? (j & 3) : t], PAIR_MASK);
                            if (j == n_kv - 1) ptx::mma_commit2_mc(&bars->o_final, PAIR_MASK);
                        }
                    }
                    __syncwarp();
                }
                if (!C::DP && j + NG < n_kv) issue_qk(j + NG);
            }
        }
    } else if (warp >= C::SM_BASE && warp < C::SM_BASE + NUM_SOFTMAX_WARPS) {
        // ------------------------------------------------------------ softmax / correction / epilogue
        ptx::setmaxnreg_inc<C::SOFTMAX_REGS>();
        const int g = (warp - C::SM_BASE) >> 2;        // softmax group: KV tiles j with j % NG == g
        const int wq = warp & 3;                       // TMEM lane quarter this warp may access (= SMSP)
        const int row = wq * 32 + lane;                // row within the tile
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tmem + lane_base + g * BN;
        const uint32_t tO = tmem + lane_base + C::O_COL;
        const float sl2 = args.scale_log2;
        const uint64_t SL2 = ptx::f2pack(sl2, sl2);
        const int last_valid = Skv_b - (n_kv - 1) * BN;   // valid keys in the last tile (1..BN)
        const bool tr = (lane == 0 && wq == 0);
        // "m of tile j-1 is in xm[]" for this warp / for the warp(s) of the next group (see Cfg::BAR_EPI)
        const uint32_t bar_in = NG == 3 ? 1 + 3 * wq + g : 1 + g;
        const uint32_t bar_out = NG == 3 ? 1 + 3 * wq + (g + 1) % NG : 1 + (g + 1) % NG;
        constexpr uint32_t BAR_N = NG == 3 ? 64 : 256;

        float mg = -INFINITY;  // the running max this group last used (its l is relative to it)
        float l = 0.f;         // this group's partial row sum (fp32)
        for (int j = g; j < n_kv; j += NG) {
            const bool masked = (j == n_kv - 1) && (last_valid < BN);
            if (tr) TRACE(j, 3);
            ptx::mbar_wait(&bars->s_full[g], (j / NG) & 1);
            ptx::tc_fence_after();
            if (tr) TRACE(j, 4);
            TRACE2(j, crank * 4 + wq, 0);
            // pass 1: row max over the BN keys, two rounds of HALF columns; with 152 registers (NG = 3) the half
            // pass 2 processes first is read second and its scores stay in registers (kv) for pass 2
            // (DP: both halves are read in one round and stay in registers; the S buffer is released right after)
            constexpr bool KEEP = NG == 3;
            constexpr bool DP = C::DP;
            float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
            uint32_t kv[HALF], ka[HALF];   // ka: DP only (the half HALF_ORDER[1])
            if (DP) {
                ptx::tmem_ld_cols<HALF>(tS + HALF * HALF_ORDER[1], ka);
                ptx::tmem_ld_cols<HALF>(tS + HALF * HALF_ORDER[0], kv);
                ptx::tmem_wait_ld();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(&bars->s_free[g], 0));   // the leader's
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int h = HALF_ORDER[1 - r];
                uint32_t tv[HALF];
                uint32_t (&sv)[HALF] = DP ? (r ? kv : ka) : ((r && KEEP) ? kv : tv);
                if (!DP) {
                    ptx::tmem_ld_cols<HALF>(tS + HALF * h, sv);
                    ptx::tmem_wait_ld();
                }
                if (masked) {
#pragma unroll
                    for (int i = 0; i < HALF; ++i)
                        if (HALF * h + i >= last_valid) sv[i] = 0xff800000u;
                }
#pragma unroll
                for (int i = 0; i < HALF; i += 8) {   // FMNMX3: two new scores per instruction, four chains
                    m0 = ptx::fmax3(m0, __uint_as_float(sv[i]), __uint_as_float(sv[i + 1]));
                    m1 = ptx::fmax3(m1, __uint_as_float(sv[i + 2]), __uint_as_float(sv[i + 3]));
                    m2 = ptx::fmax3(m2, __uint_as_float(sv[i + 4]), __uint_as_float(sv[i + 5]));
                    m3 = ptx::fmax3(m3, __uint_as_float(sv[i + 6]), __uint_as_float(sv[i + 7]));
                }
            }
            const float mx = ptx::fmax3(m0, m1, fmaxf(m2, m3)) * sl2;
            if (tr) TRACE(j, 7);
            // running max after tile j-1, handed over by the previous group (strict tile order)
            float mprev = -INFINITY;
            if (j > 0) {
                ptx::named_bar_sync(bar_in, BAR_N);
                mprev = xm[row];
            }
            const bool resc = mx > mprev + RESCALE_TAU;   // also true on tile 0 (mprev = -inf)
            const float m = resc ? mx : mprev;
            if (j + 1 < n_kv) {
                xm[row] = m;
                __threadfence_block();
                ptx::named_bar_arrive(bar_out, BAR_N);
            }
            if (tr) TRACE(j, 5);
            if (m != mg) {   // this group's partial sum follows the reference max
                l *= ptx::ex2(mg - m);   // mg = -inf: l = 0 anyway
                mg = m;
            }
            if (j > 0 && __any_sync(0xffffffffu, resc)) {
                // O *= 2^(mprev - m) for the moved rows (others by exactly 1), after PV(j-1), the last product
                // into O, completed; PV(j) waits for this P.
                const float factor = resc ? ptx::ex2(mprev - m) : 1.f;
                // PV(j-1) is completion jp/NG of pv_done[jp%NG].  The parity test is unambiguous: PV(j-1-NG) was
                // committed before S(j-1), which the previous group saw complete before handing over the max,
                // and PV(j-1+NG) cannot complete before PV(j), which needs this group's P(j).
                const int jp = j - 1;
                // (DP: PV(j) completes on pv_done[j % 4]; PV(j-5) completed before S(j), so the parity is unambiguous)
                if (DP) ptx::mbar_wait(&bars->pv_done[jp & 3], (jp >> 2) & 1);
                else ptx::mbar_wait(&bars->pv_done[jp % NG], (jp / NG) & 1);
                ptx::tc_fence_after();
                constexpr int RC = DP ? 16 : 32;   // columns per round (DP holds 2 x HALF scores in registers)
#pragma unroll
                for (int c = 0; c < D / RC; ++c) {
                    uint32_t r[RC];
                    ptx::tmem_ld_cols<RC>(tO + RC * c, r);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < RC; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * factor);
                    ptx::tmem_st_cols<RC>(tO + RC * c, r);
                }
            }
            // pass 2, per HALF-key half: P = exp2(s*sl2 - m) in f32x2 pairs (MUFU or FMA-pipe polynomial by
            // column), bf16 pairs written over the half's first HALF/2 score columns (already read), released to
            // the MMA issuer.
            const uint64_t NEGM = ptx::f2pack(-m, -m);
            uint64_t L0 = ptx::f2pack(0.f, 0.f), L1 = L0;
            if (DP && j >= 2) {   // P buffer j % 2 is free once PV(j-2) completed (PV(j-6) did before S(j))
                ptx::mbar_wait(&bars->pv_done[(j - 2) & 3], ((j - 2) >> 2) & 1);
                ptx::tc_fence_after();
            }
            const uint32_t tP = DP ? tmem + lane_base + C::P_COL + (j & 1) * HALF : tS;
#pragma unroll
            for (int o = 0; o < 2; ++o) {
                const int h = HALF_ORDER[o];
                uint32_t tv[HALF];
                // KEEP: the first half is still in registers; DP: both are
                uint32_t (&sv)[HALF] = DP ? (o ? ka : kv) : ((o || !KEEP) ? tv : kv);
                if ((o || !KEEP) && !DP) {
                    ptx::tmem_ld_cols<HALF>(tS + HALF * h, sv);
                    ptx::tmem_wait_ld();
                    if (masked) {
#pragma unroll
                        for (int i = 0; i < HALF; ++i)
                            if (HALF * h + i >= last_valid) sv[i] = 0xff800000u;
                    }
                }
                uint32_t pk[HALF / 2];
#pragma unroll
                for (int i = 0; i < HALF / 2; ++i) {
                    const int e = 2 * i;
                    const uint64_t X =
                        ptx::ffma2(ptx::f2pack(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), SL2, NEGM);
                    float p0, p1;
                    if ((e & 15) >= C::POLY_FROM) {
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
                ptx::tmem_st_cols<HALF / 2>(tP + (DP ? HALF / 2 : HALF) * h, pk);
                ptx::tmem_wait_st();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(&bars->p_full[DP ? (j & 1) : g][h], 0));   // the leader's
                if (tr && o == 0) TRACE(j, 8);
                TRACE2(j, crank * 4 + wq, 1 + o);
            }
            {
                float a0, a1, b0, b1;
                ptx::f2unpack(L0, a0, a1);
                ptx::f2unpack(L1, b0, b1);
                l += (a0 + b0) + (a1 + b1);
            }
            if (tr) TRACE(j, 6);
        }
        // ------------------------------------------------------------ epilogue: merge group sums, O / l -> global
        if (n_kv > 0) {
            ptx::mbar_wait(&bars->o_final, 0);   // ring slot 0 is idle from here on (see xml)
            ptx::tc_fence_after();
        }
        xml[g][row] = mg;
        xml[NG + g][row] = l;
        ptx::named_bar_sync(C::BAR_EPI, 32 * NUM_SOFTMAX_WARPS);
        float mm = -INFINITY;
#pragma unroll
        for (int q = 0; q < NG; ++q) mm = fmaxf(mm, xml[q][row]);   // = the max after the last tile, O's reference
        float lsum = 0.f;
#pragma unroll
        for (int q = 0; q < NG; ++q) {
            const float mq = xml[q][row];
            if (mq != -INFINITY) lsum += xml[NG + q][row] * ptx::ex2(mq - mm);   // a group may have no tile
        }
        const float inv = n_kv > 0 ? 1.f / lsum : 0.f;   // no valid key: the row is 0 (R20)
        const long long srow = (long long)qtile * BM + row;
        const bool valid = srow < args.Sq;      // tcgen05.ld is warp-collective: every lane loads, valid lanes store
        const long long oidx = (long long)b * args.o_batch_stride + srow * args.o_tok_stride + (long long)head * D;
        uint4 *dst = reinterpret_cast<uint4 *>(args.O + oidx);
        if (args.n_dst > 0) {   // direct transport: this row belongs to source rank i's output buffer
            int i = 0;
            while (i + 1 < args.n_dst && srow >= args.row_begin[i + 1]) ++i;
            dst = reinterpret_cast<uint4 *>(args.dst[i] + (long long)b * args.dst_batch_stride[i] +
                                            (srow - args.row_begin[i]) * args.o_tok_stride + (long long)head * D);
        }
        // ring / merge support: the row's log-sum-exp of the scaled scores, ln sum_t exp(q.k_t / sqrt(D)) =
        // (running max + log2 l) * ln 2 in the kernel's base-2 domain; -inf for a row without valid keys
        if (args.lse && valid && g == 0)
            args.lse[((long long)b * args.Sq + srow) * args.lse_heads + head] =
                n_kv > 0 ? (mm + __log2f(lsum)) * 0.69314718055994531f : -INFINITY;
        // this warp normalises and stores the 16-column chunks c with c % NG == g
#pragma unroll
        for (int c = 0; c < C::OCHUNKS; ++c) {
            if (c % NG != g) continue;
            const int col = 16 * c;
            uint32_t r[16];
            if (n_kv > 0) {
                ptx::tmem_ld16(tO + col, r);
                ptx::tmem_wait_ld();
            } else {
#pragma unroll
                for (int u = 0; u < 16; ++u) r[u] = 0u;
            }
            if (args.O32) {   // fp32 output (partial results of ring attention, merged by spa_lse_merge)
                if (valid) {
                    float4 *d4 = reinterpret_cast<float4 *>(args.O32 + oidx + col);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        d4[u] = make_float4(__uint_as_float(r[4 * u]) * inv, __uint_as_float(r[4 * u + 1]) * inv,
                                            __uint_as_float(r[4 * u + 2]) * inv, __uint_as_float(r[4 * u + 3]) * inv);
                }
                continue;
            }
            uint32_t w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                w[u] = ptx::pack_bf16x2(__uint_as_float(r[2 * u]) * inv, __uint_as_float(r[2 * u + 1]) * inv);
            if (valid) {
                dst[col / 8] = make_uint4(w[0], w[1], w[2], w[3]);
                dst[col / 8 + 1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
        }
    } else {
        ptx::setmaxnreg_dec<C::AUX_REGS>();   // idle warps of the last warpgroup
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();   // no CTA leaves while its peer may still signal its barriers or read its smem / TMEM
    if (warp == MMA_WARP) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc2(tmem, C::TMEM_COLS);
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
// swz = swizzle width in bytes (32, 64 or 128) = the UMMA layout the box lands in.
bool make_map(CUtensorMap *m, const void *base, int D, int heads, int S, int B, long long tok_stride,
              long long batch_stride, int box_d, int swz, int box_rows = BM) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)heads, (cuuint64_t)S, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)tok_stride * 2, (cuuint64_t)batch_stride * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_d, 1, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : (swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B),
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int D>
cudaError_t launch_d(const AttnProblem &p, cudaStream_t st) {
    using C = Cfg<D>;
    // m[0]/m[1]: Q 64-col SW128 / 32-col SW64 boxes of 128 rows; m[2]/m[3]: the same for K with 64-row boxes
    // (a CTA's half of a K tile); m[4]: V boxes of one swizzle atom (64 / 32 / 16 columns for D = 128 / 64 / 96)
    // by 128 rows (a CTA's half of a V tile is D/2 columns); m[5] unused.
    CUtensorMap m[6];
    const int vswz = C::V_ATOM_COLS * 2;
    bool ok = make_map(&m[0], p.q, D, p.n_heads, p.Sq, p.B, p.q_tok_stride, p.q_batch_stride, 64, 128) &&
              make_map(&m[2], p.k, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, 64, 128, C::BN / 2) &&
              make_map(&m[4], p.v, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, C::V_ATOM_COLS, vswz,
                       C::BN);
    if (ok && C::N64)
        ok = make_map(&m[1], p.q, D, p.n_heads, p.Sq, p.B, p.q_tok_stride, p.q_batch_stride, 32, 64) &&
             make_map(&m[3], p.k, D, p.n_heads, p.Skv, p.B, p.kv_tok_stride, p.kv_batch_stride, 32, 64, C::BN / 2);
    else {
        m[1] = m[0];
        m[3] = m[2];
    }
    m[5] = m[4];
    if (!ok) return cudaErrorInvalidValue;
    // The smem opt-in is a per-device (per-context) function attribute: set it once per device, thread-safely.
    static std::atomic<uint64_t> attr_done{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_done.fetch_or(bit, std::memory_order_release);
    }
    AttnArgs a;
    a.O = reinterpret_cast<__nv_bfloat16 *>(p.o);
    a.o_tok_stride = p.o_tok_stride;
    a.o_batch_stride = p.o_batch_stride;
    a.Sq = p.Sq;
    a.Skv = p.Skv;
    a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
    a.kv_len = p.kv_len;
    a.kv_offset = p.kv_offset;
    a.O32 = reinterpret_cast<float *>(p.o32);
    a.lse = p.lse;
    a.lse_heads = p.n_heads;
    a.n_dst = p.n_dst;
    for (int i = 0; i < kMaxDst; ++i) {
        a.dst[i] = reinterpret_cast<__nv_bfloat16 *>(p.dst[i]);
        a.dst_batch_stride[i] = p.dst_batch_stride[i];
        a.row_begin[i] = p.row_begin[i];
    }
    a.row_begin[kMaxDst] = p.row_begin[kMaxDst];
    // CTA pairs (adjacent query tiles of one head) run each MMA as one cta_group::2 instruction; an odd tile
    // count gets one extra all-out-of-range tile (zero-filled Q, rows never stored) to complete the last pair.
    const int qtiles = (p.Sq + BM - 1) / BM;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((qtiles + 1) / 2 * 2, p.n_heads, p.B);
    cfg.blockDim = dim3(C::NUM_THREADS);
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
extern "C" int spa_debug_read_trace2(unsigned long long *out) {
    return (int)cudaMemcpyFromSymbol(out, g_trace2, sizeof(g_trace2));
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
