/*
 * spa.h -- C ABI of the B200-native PipeSP sequence-parallel attention library
 * (libspa.so, built from paper_2511_12056_b200/csrc/).
 *
 * What the library computes (PAPER.md = /root/reference/PAPER.md):
 *   Each of P ranks holds a sequence shard Q_r, K_r, V_r of shape [B, S/P, H, D]
 *   (bf16, contiguous).  Every rank receives its sequence shard of
 *       O = softmax(Q K^T / sqrt(D)) V        per batch b and head k,
 *   i.e. O[:, r*S/P:(r+1)*S/P, :, :] in the same [B, S/P, H, D] layout.
 *   - Ulysses SP (Fig. 3(a)): seq->head all-to-all of Q, K, V,
 *     attention over the full sequence on H/P local heads, head->seq all-to-all.
 *   - PipeSP (Alg. 1): the same result, with the attention split
 *     into N_st pipeline stages; stage k's output all-to-all (and stage k+1's input
 *     all-to-all) overlap stage k+1's (k's) attention.  The paper's per-head order
 *     fix view->permute->view (proof PAPER.md:516-578) is fused
 *     into the final gather, so the interleaved layout is never materialised.
 *   - Aco (Fig. 4): attention of the heads is spread over
 *     N_src "denoising" ranks plus spare "decoding" ranks; only source ranks hold
 *     input and output shards.
 *   The softmax scale 1/sqrt(D) is the north star's (the paper never states it).
 *
 * Numerics: bf16 inputs, fp32 QK^T accumulation and fp32 online softmax, P rounded
 * to bf16 for the PV product, fp32 O accumulation, bf16 (RNE) output.  Tolerance
 * vs the fp64 definition: max-abs 2e-2 and rel-L2 5e-3 (BASELINE.json north_star).
 * The resharding steps are pure permutations: bit-exact.
 *
 * Conventions
 *   - All functions return spa_status; SPA_OK == 0.  Argument / shape errors are
 *     detected synchronously and NOTHING is enqueued.  spa_last_error() returns a
 *     thread-local message for the last failing call on this thread.
 *   - Device pointers: 16-byte aligned, caller-owned (e.g. torch tensors).  The
 *     library owns comms, plans, its comm stream and events.
 *   - Stream-ordered: work is enqueued after prior work on `stream` and the output
 *     is valid when `stream` reaches the end of the call; inputs must not be
 *     modified before that.  Calls return as soon as everything is enqueued.
 *   - Collective: with an NCCL comm every rank must call with identical plans in the
 *     same order (like NCCL itself).
 *   - Determinism: identical inputs give bit-identical outputs, for any rank count
 *     and any stage count (each output row depends only on its own query row and
 *     the full K/V of its head, evaluated in a fixed key-tile order).
 *   - Not thread-safe per plan: one call at a time per plan.
 */
#ifndef SPA_H_
#define SPA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPA_OK = 0,
    SPA_ERR_INVALID = 1,     /* null pointer, bad enum, misaligned pointer, wrong comm kind */
    SPA_ERR_SHAPE = 2,       /* S < n_src, H % n_owners != 0, stages < 1, query chunks > shortest shard */
    SPA_ERR_UNSUPPORTED = 3, /* D not in {64, 96, 128}, op not available on this comm kind */
    SPA_ERR_CUDA = 4,        /* CUDA runtime/driver error (incl. a previous async kernel fault) */
    SPA_ERR_COMM = 5,        /* NCCL error or async communicator failure */
    SPA_ERR_BUSY = 6         /* Aco co-processor group busy: caller falls back to PipeSP */
} spa_status;

typedef struct spa_comm spa_comm; /* rank group ("RankGroup") */
typedef struct spa_plan spa_plan;

/* ------------------------------------------------------------------ rank groups */
/* NCCL unique id (128 bytes) created on rank 0; the caller broadcasts it (torch.distributed). */
spa_status spa_get_unique_id(uint8_t id[128]);
/* One process per GPU: NCCL communicator of `nranks` ranks over NVLink/NVSwitch; `device` = CUDA ordinal.
 * Validation status: the NCCL message lists are matched across ranks on the host and exchanged over
 * gloo, a 1-rank NCCL communicator runs on the GPU; the multi-GPU NCCL exchange itself has not run in this build's
 * one-GPU test environment -- the P2P transport (spa_comm_init_p2p) has, with real processes. */
spa_status spa_comm_init(spa_comm **comm, const uint8_t id[128], int nranks, int rank, int device);
/* The same with NCCL communicator settings: the SM budget of NCCL's kernels while the attention grid occupies the
 * GPU (ncclConfig_t minCTAs / maxCTAs / CTAPolicy; NCCL 2.28).  0 leaves a field at NCCL's default (and its env
 * variables, e.g. NCCL_MAX_CTAS, apply).  cta_policy: 0 default, 1 efficiency, 2 zero-CTA (copy engines, for
 * buffers NCCL supports it on). */
typedef struct {
    int min_ctas, max_ctas, cta_policy;
} spa_comm_config;
spa_status spa_comm_init_config(spa_comm **comm, const uint8_t id[128], int nranks, int rank, int device,
                                const spa_comm_config *cfg);
/* Failure handling: waits until `stream` completes, polling the communicator's asynchronous error state.  A peer
 * failure (NCCL async error) or no completion within timeout_ms (< 0: no limit) ABORTS the NCCL communicator
 * (ncclCommAbort unblocks this rank's pending NCCL kernels) and returns SPA_ERR_COMM; the comm can then only be
 * destroyed.  Returns SPA_OK when the stream completed, SPA_ERR_CUDA on a CUDA fault. */
spa_status spa_comm_wait(spa_comm *comm, void *stream, int timeout_ms);
/* `nvirtual` virtual ranks on ONE GPU (tests / single-GPU measurement): the all-to-all
 * becomes device-to-device copies on the comm stream, everything else is identical. */
spa_status spa_comm_init_loopback(spa_comm **comm, int nvirtual, int device);
/* One process per GPU WITHOUT NCCL: the exchange runs over CUDA IPC peer memory (NVLink / NVSwitch between GPUs;
 * also valid for several processes sharing one GPU) -- SURVEY f1, DESIGN.md §6.  Every rank's workspace is mapped
 * into every other rank (spa_plan_ipc_handle / spa_plan_ipc_open below); the staged exchange is copy-engine
 * cudaMemcpyAsync of each message straight into the receiver's region (no SMs taken from the attention), and
 * SPA_OPT_DIRECT makes the pack kernel and the attention epilogue store to the peers themselves.  Cross-process
 * order: per-call epoch flags in each workspace's tail, written with cuStreamWriteValue32 (system-scope fence
 * first) after the data and awaited with cuStreamWaitValue32 -- no kernel ever spins on a flag.  Ulysses / PipeSP /
 * Aco / QKV / Ring / USP plans and the reshard calls (the ring's K/V blocks travel by copy engine into the next
 * rank's receive slot, with arrival and slot-free flags; a USP plan's Ulysses and ring sub-groups are mapped by its
 * own spa_plan_ipc_open).  `rank` and `nranks` come from the caller's launcher. */
spa_status spa_comm_init_p2p(spa_comm **comm, int nranks, int rank, int device);
/* Host-only rank group: plans can be created, validated and described (spa_plan_describe_*),
 * but not executed.  Used to test the multi-rank host logic without a GPU. */
spa_status spa_comm_init_host(spa_comm **comm, int nranks, int rank);
/* Sub-group (e.g. the denoising group for Aco's busy fallback): ranks with the same
 * color form a group ordered by key; color < 0 -> *sub = NULL.  NCCL: ncclCommSplit. */
spa_status spa_comm_split(spa_comm *comm, int color, int key, spa_comm **sub);
/* Polls the communicator for asynchronous errors (NCCL async error / CUDA sticky error). */
spa_status spa_comm_check(spa_comm *comm);
spa_status spa_comm_destroy(spa_comm *comm);
/* rank count / own rank (-1 for loopback, which holds all ranks). */
spa_status spa_comm_info(const spa_comm *comm, int *nranks, int *rank, int *kind /* 0 nccl,1 loopback,2 host,3 p2p */);

/* ------------------------------------------------------------------ plans */
typedef struct {
    int B, S, H, D; /* global problem: batch, sequence length, heads, head dim (bf16) */
    int stages;     /* N_st pipeline stages (R7): G_h = gcd(N_st, h) head groups of
                       g = h/G_h heads, C = N_st/G_h query chunks; 1 = Ulysses (one stage) */
    int n_src;      /* ranks holding sequence shards: 0 = all ranks (Ulysses/PipeSP);
                       0 < n_src < nranks = Aco (ranks >= n_src are co-processors) */
    int pad_heads;  /* 0: H % nranks must be 0.  1: head padding ("padding increases
                       the head count to 28 so that each GPU handles 4 heads"): the heads are padded to
                       Hp = spa_pad_heads(H, nranks); rank r owns padded heads [r*Hp/nranks, (r+1)*Hp/nranks);
                       pad heads are never read from q/k/v, never computed and never written to out
                       (user buffers keep H heads).  DESIGN.md R10. */
    int ring;       /* 0: Ulysses / PipeSP / Aco plan.  1: Ring-Attention plan ("switch ... from
                       Ulysses to Ring-Attention ... avoiding the overhead of padding"; R21): every
                       rank keeps all H heads of its sequence shard, only S % nranks == 0 is required (any H);
                       use spa_ring_attention*.  stages must be 1 and pad_heads 0 (else SPA_ERR_INVALID);
                       n_src 0 or nranks (else SPA_ERR_SHAPE). */
    int ulysses;    /* ring plans only: Ulysses degree U of the USP hybrid ("flexible configuration
                       of both the Ulysses degree and the Ring-Attention degree"); 0 or 1 = pure Ring.  U > 1:
                       U | nranks and U | H; ranks [rho*U, rho*U+U) form Ulysses group rho, the R = nranks/U
                       groups form rings (seq->head all-to-all in the group, Ring attention over the groups on
                       H/U heads, head->seq all-to-all).  NCCL plans split the comm (plan creation is then
                       collective). */
} spa_shape;

/* Validates everything synchronously.  Sequence shards: source rank r holds tokens [start_r, start_r + len_r)
 * with len_r = S/n_src + (r < S % n_src ? 1 : 0) -- equal when n_src divides S, otherwise differing by one
 * token (R9; e.g. Aco with 7 denoising GPUs); q, k, v, out of rank r have len_r
 * tokens.  Requirements: D in {64,96,128}; S >= n_src; (ring / USP plans: S % nranks == 0);
 * H % nranks == 0 unless pad_heads (heads are split over ALL ranks, which own contiguous head blocks);
 * 1 <= stages and C <= S/n_src (C and G_h follow from h = Hp/nranks). */
spa_status spa_plan_create(spa_plan **plan, spa_comm *comm, const spa_shape *shape);
/* Device workspace bytes the caller must pass as `ws` (per rank; for loopback plans:
 * for all virtual ranks together).  Zero when nranks == 1. */
spa_status spa_plan_workspace_bytes(const spa_plan *plan, size_t *bytes);
/* P2P plans (spa_comm_init_p2p): register the workspace the calls will pass (device memory of at least
 * spa_plan_workspace_bytes(); e.g. a torch tensor).  Collective set-up, once per plan:
 *   1. every rank: spa_plan_ipc_handle(plan, ws, handle)   -- SPA_IPC_HANDLE_BYTES bytes (CUDA IPC handle of the
 *      allocation holding ws + the offset of ws in it)
 *   2. the caller gathers all ranks' handles in rank order (e.g. torch.distributed.all_gather_object)
 *   3. every rank: spa_plan_ipc_open(plan, ws, handles)    -- maps the peers' workspaces, zeroes this rank's flags
 *   4. a host barrier over all ranks (so that no flag is written before its owner zeroed it)
 * Afterwards every call must pass this same ws; spa_plan_destroy unmaps the peers. */
#define SPA_IPC_HANDLE_BYTES 72
spa_status spa_plan_ipc_handle(spa_plan *plan, void *ws, uint8_t handle[SPA_IPC_HANDLE_BYTES]);
spa_status spa_plan_ipc_open(spa_plan *plan, void *ws, const uint8_t *handles);
/* NCCL plans on NCCL symmetric-memory windows (NCCL >= 2.28; SURVEY f1 on NVLink / NVSwitch): the exchange then
 * runs on peer memory exactly as for P2P plans -- copy-engine copies of every message straight into the receivers'
 * regions, or with SPA_OPT_DIRECT the pack kernel's and the attention epilogue's stores into the peers -- ordered by
 * the same per-call epoch flags, instead of NCCL send / recv.  Set-up, once per plan:
 *   1. every rank: spa_mem_alloc(bytes, &ws) with bytes >= spa_plan_workspace_bytes(plan) rounded up to 4096
 *      (ncclMemAlloc: the memory NCCL can map into its peers)
 *   2. every rank: spa_plan_window_register(plan, ws) -- COLLECTIVE over the plan's communicator
 *      (ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC); resolves every rank's address of its window with NCCL's
 *      device API (ncclGetLsaPointer) and zeroes this rank's flags.  SPA_ERR_UNSUPPORTED if the communicator's LSA
 *      team (ncclDevCommCreate: the ranks NCCL maps into each other, one NVLink domain) is not all ranks; SPA_ERR_UNSUPPORTED for ring / USP plans (they keep NCCL send / recv); 1-rank plans: no-op.
 *   3. a host barrier over all ranks before the first call
 * Afterwards every call passes this ws; spa_plan_destroy deregisters the window; spa_mem_free(ws) after that.
 * SPA_OPT_DIRECT on an NCCL plan requires the window (SPA_ERR_INVALID at the call otherwise).  Validation status:
 * the peer-memory execution is the P2P transport's (multi-process tested); the window plumbing is checked on one
 * GPU by spa_comm_window_selftest; an NCCL exchange between several GPUs has not run in this build's environment. */
spa_status spa_mem_alloc(size_t bytes, void **ptr);
spa_status spa_mem_free(void *ptr);
spa_status spa_plan_window_register(spa_plan *plan, void *ws);
/* One-GPU check of the window plumbing on an NCCL comm (collective): ncclMemAlloc `bytes` (a multiple of 4096),
 * register them as a symmetric window, resolve every rank's LSA address on the device, store a pattern through THIS
 * rank's LSA address with a kernel and read it back through the local pointer; SPA_OK iff every word matches. */
spa_status spa_comm_window_selftest(spa_comm *comm, size_t bytes);
/* G_h, C, g of the plan's stage split. */
spa_status spa_plan_stage_split(const spa_plan *plan, int *G_h, int *C, int *g);
spa_status spa_plan_destroy(spa_plan *plan);

/* Measurement knobs (bench only; never change results except SKIP_COMM).
 *   SPA_OPT_PROFILE   1 -> record CUDA events around every step of the next calls
 *   SPA_OPT_SKIP_COMM 1 -> the all-to-alls are not issued (exposed-comm measurement;
 *                          the output is then NOT the attention result)
 *   SPA_OPT_COPROC_BUSY 1 -> the decoding group is busy (Fig. 4 prompt-2 stage): spa_aco_*
 *                          return SPA_ERR_BUSY without enqueueing; the caller runs PipeSP on
 *                          the denoising sub-group instead */
/*   SPA_OPT_DIRECT    1 -> direct transport: the pack stores straight into the
 *                          owners' receive regions and the attention epilogue stores each output row straight
 *                          into its source rank's output (no staging, exchange copies or unpack).  Loopback
 *                          plans, P2P plans, and NCCL plans with a registered window (spa_plan_window_register);
 *                          same bits. */
/*   SPA_OPT_COMM_SMS  n -> the persistent QKV-projection GEMM (spa_pipesp_qkv_attention*) leaves n SMs free so that
 *                          the communication kernels of the overlapped all-to-alls get SMs at once (0..64; default 0) */
/*   SPA_OPT_RANK_ONLY r+1 -> loopback plans: only virtual rank r's launches and the messages it sends or receives
 *                          run (0 = all ranks) -- one rank's share of the multi-GPU schedule measured on one GPU
 *                          (wave tails, copy/attention SM contention); the output is then NOT the attention result
 *   SPA_OPT_LOOPBACK_CE 1 -> loopback exchange messages as copy-engine cudaMemcpyAsync (the P2P transport's staged
 *                          exchange) instead of the copy kernel (NCCL-like: SMs move the bytes); same result bits */
/*   SPA_OPT_STAGE_WINDOW w -> up to w pipeline stages in flight (1..8, default 4): their attention launches go to w
 *                          compute streams round-robin and the input exchange runs w stages ahead; wider windows keep
 *                          the GPU full when stages are small (many stages of a short sequence); same result bits */
enum { SPA_OPT_PROFILE = 1, SPA_OPT_SKIP_COMM = 2, SPA_OPT_COPROC_BUSY = 3, SPA_OPT_DIRECT = 4, SPA_OPT_COMM_SMS = 5,
       SPA_OPT_RANK_ONLY = 6, SPA_OPT_LOOPBACK_CE = 7, SPA_OPT_STAGE_WINDOW = 8 };
spa_status spa_plan_set_option(spa_plan *plan, int option, int value);

/* Key-padding mask for the following SP calls of this plan (Alg. 1's attention_mask, PAPER.md:85 and :90,
 * which the paper never defines -- DESIGN.md reading R20): kv_len = device int32 [B]; key t of batch entry b
 * (global sequence position, 0 <= t < S) takes part in the softmax iff t < kv_len[b] (values clamped to
 * [0, S]); a batch entry with kv_len 0 gives output rows of 0.  Query rows are never masked.  NULL clears
 * the mask.  The array is read by the kernels when they run (stream-ordered): it must stay valid and
 * unchanged until the calls' streams complete.  NCCL plans: each rank passes its own device copy.
 * Masked key tiles are skipped entirely (work scales with kv_len). */
spa_status spa_plan_set_kv_len(spa_plan *plan, const int32_t *kv_len);

/* Per-step device times (ms) of the last profiled call, once its stream has completed.
 * attn_ms[k], a2a_in_ms[k], a2a_out_ms[k] for k < n_stages (arrays of >= 64 entries). */
typedef struct {
    int n_stages;
    float total_ms;   /* whole call, first to last event on the caller's stream */
    float pack_ms, unpack_ms;
    float attn_ms[64], a2a_in_ms[64], a2a_out_ms[64];
    int attn_launches, copy_launches; /* library kernels launched by the call */
    int gemm_launches;                /* QKV-projection GEMMs (pack_ms is then the projection time) */
} spa_profile;
spa_status spa_plan_last_profile(spa_plan *plan, spa_profile *out);

/* ------------------------------------------------------------------ SP attention (per-rank collective calls)
 * q, k, v, out: device bf16 [B, S/n_src, H, D] contiguous (this rank's shard); ws: device
 * workspace of spa_plan_workspace_bytes(); stream: cudaStream_t of the caller.
 * NCCL or P2P plans (loopback plans use the *_local variants). */
spa_status spa_ulysses_attention(spa_plan *plan, const void *q, const void *k, const void *v, void *out,
                                 void *ws, void *stream);
spa_status spa_pipesp_attention(spa_plan *plan, const void *q, const void *k, const void *v, void *out,
                                void *ws, void *stream);
/* Aco: plan with 0 < n_src < nranks.  Ranks < n_src pass their shards;
 * co-processor ranks (>= n_src) pass NULL for q, k, v, out.  A plan without co-processor ranks
 * (n_src == 0 or nranks, i.e. N_decode = 0) runs PipeSP on all ranks. */
spa_status spa_aco_attention(spa_plan *plan, const void *q, const void *k, const void *v, void *out,
                             void *ws, void *stream);

/* Loopback plans: arrays with one pointer per source rank (n_src entries, or nranks when
 * n_src == 0); all virtual ranks are enqueued on `stream`. */
spa_status spa_ulysses_attention_local(spa_plan *plan, const void *const q[], const void *const k[],
                                       const void *const v[], void *const out[], void *ws, void *stream);
spa_status spa_pipesp_attention_local(spa_plan *plan, const void *const q[], const void *const k[],
                                      const void *const v[], void *const out[], void *ws, void *stream);
spa_status spa_aco_attention_local(spa_plan *plan, const void *const q[], const void *const k[],
                                   const void *const v[], void *const out[], void *ws, void *stream);

/* Single-GPU attention from and to HOST memory (pinned for overlap; 1-rank loopback plan): q, k, v, o are host
 * [B, S, H, D] bf16; ws = device workspace of spa_plan_host_workspace_bytes() (device copies of Q, K, V, O).
 * The plan's `stages` sets the head-group count G_h = gcd(stages, H): the H2D copy of group i+1's columns
 * and the D2H copy of group i-1's output overlap group i's attention (two extra streams; the output is in
 * `o` when `stream` reaches the end of the call).  Same result bits as spa_attention_fwd on those heads. */
spa_status spa_plan_host_workspace_bytes(const spa_plan *plan, size_t *bytes);
spa_status spa_attention_host(spa_plan *plan, const void *q, const void *k, const void *v, void *o, void *ws,
                              void *stream);

/* The SP layer (spa_pipesp_attention) from and to HOST memory at any rank count (pinned host buffers for overlap):
 * q, k, v, out = host [B, S_r, H, D] bf16 of this rank (loopback: one per source rank; Aco co-processor ranks pass
 * NULL); ws = spa_plan_host_sp_workspace_bytes(): the plan's workspace followed by device copies of the local Q, K, V,
 * O.  Per head group kh of the stage split: the H2D of its heads' columns (for every destination rank) runs on a copy
 * stream and only group kh's pack waits for it; as soon as the last stage of group kh is exchanged back, its unpack
 * and the D2H of its output columns run on a second copy stream -- the copies overlap the other groups' exchange and
 * attention.  Same result bits as spa_pipesp_attention.  1-rank plans: spa_attention_host.  P2P plans: register this
 * ws (spa_plan_ipc_handle / open).  Not for ring plans; SPA_OPT_DIRECT does not apply. */
spa_status spa_plan_host_sp_workspace_bytes(const spa_plan *plan, size_t *bytes);
spa_status spa_pipesp_attention_hostbuf(spa_plan *plan, const void *q, const void *k, const void *v, void *out,
                                        void *ws, void *stream);
spa_status spa_pipesp_attention_hostbuf_local(spa_plan *plan, const void *const q[], const void *const k[],
                                              const void *const v[], void *const out[], void *ws, void *stream);

/* ------------------------------------------------------------------ QKV projection fused with PipeSP
 * The SP layer from the hidden states ("after each GPU computes its portion of the sub-sequence's
 * Q, K, and V, three rounds of All-to-All ..."; the projections Q = X W_Q, K = X W_K, V = X W_V of PAPER.md:155-157,
 * overlapped with the input all-to-alls as in PAPER.md:439).  Per head group kh of the plan's stage split, one
 * tcgen05 GEMM computes this rank's X [B, S_r, C] times the head group's weight rows for EVERY destination rank and
 * stores the result (fp32 accumulate + fp32 bias, bf16 RNE) straight into the stage's all-to-all send layout (the
 * pack step is fused away); head group kh's input all-to-all then overlaps head group kh+1's GEMM, and the rest is
 * spa_pipesp_attention.  Plans: Ulysses / PipeSP (n_src = 0, no head padding, no ring).  With SPA_OPT_DIRECT each
 * head group's GEMM stores its columns straight into every owner's receive regions (loopback: the virtual ranks'
 * workspaces; P2P / NCCL-window plans: the peers' over NVLink; Q rows into their query chunk's stage, up to 32 chunks)
 * -- projection, pack and input all-to-all in one kernel -- and flags the group's stages to the owners; same bits.  Result = spa_pipesp_attention on bf16(X W^T + b), bit for bit.
 *
 *   w      bf16 [3*H*D, C], the fused nn.Linear weight: output feature o = t*H*D + k*D + d (t = 0 Q, 1 K, 2 V;
 *          head k; dim d).  bias: fp32 [3*H*D] or NULL.  C: hidden dim, a positive multiple of 8.
 *   w_packed  device buffer of spa_plan_qkv_weight_bytes(plan, C) bytes, written by spa_plan_pack_qkv_weight
 *          (once per plan and weight; it depends on the plan's P and stage split): the weight rows of each head group
 *          in [t][dest q][g*D] order followed by the bias in the same order as fp32.
 *   x      bf16 [B, S_r, C] contiguous (this rank's sequence shard of the hidden states; loopback: one per rank).
 *   ws     spa_plan_qkv_workspace_bytes(): spa_plan_workspace_bytes() when nranks > 1; the projected Q, K, V
 *          [B, S, H, D] when nranks == 1. */
spa_status spa_plan_qkv_weight_bytes(const spa_plan *plan, int C, size_t *bytes);
spa_status spa_plan_qkv_workspace_bytes(const spa_plan *plan, size_t *bytes);
spa_status spa_plan_pack_qkv_weight(spa_plan *plan, int C, const void *w, const float *bias, void *w_packed,
                                    void *stream);
spa_status spa_pipesp_qkv_attention(spa_plan *plan, int C, const void *x, const void *w_packed, void *out, void *ws,
                                    void *stream);
spa_status spa_pipesp_qkv_attention_local(spa_plan *plan, int C, const void *const x[], const void *w_packed,
                                          void *const out[], void *ws, void *stream);
/* The projections alone, in the standard layout: q, k, v = bf16 [B, S_r, H, D] of source rank `rank` (its x is
 * [B, S_r, C]; NCCL plans: rank must be the comm's own).  Same GEMM and rounding as the fused calls, so
 * spa_pipesp_attention on these q, k, v equals spa_pipesp_qkv_attention bit for bit. */
spa_status spa_qkv_projection(spa_plan *plan, int C, int rank, const void *x, const void *w_packed, void *q, void *k,
                              void *v, void *stream);

/* Ring attention (shape.ring = 1; R21): q, k, v, out as above ([B, S/P, H, D], any H).  Rank r
 * attends to the K/V shard of rank (r - t) mod P at step t; the shards travel the ring r-1 -> r -> r+1 on
 * the comm stream (double-buffered, NCCL send/recv) while the previous block is computed; each step writes
 * an fp32 partial result and its per-row log-sum-exp into ws, and a merge kernel combines the P partials
 * (softmax over the union of the blocks).  Not bit-identical to the Ulysses path (a different summation
 * order), within the same tolerance of the fp64 definition.  Key-padding masks (spa_plan_set_kv_len) apply by
 * global key position to every block (a wholly masked block contributes lse = -inf). */
spa_status spa_ring_attention(spa_plan *plan, const void *q, const void *k, const void *v, void *out, void *ws,
                              void *stream);
spa_status spa_ring_attention_local(spa_plan *plan, const void *const q[], const void *const k[],
                                    const void *const v[], void *const out[], void *ws, void *stream);

/* ------------------------------------------------------------------ building blocks (bit-exact tests)
 * seq->head reshard ("all_to_all"): x [B,S/P,H,D] ->
 * x_head [B,S,h,D] where x_head[b, p*S/P+t, j] = x_p[b, t, rank*h+j].  One stage. */
spa_status spa_reshard_seq_to_head(spa_plan *plan, const void *x, void *x_head, void *ws, void *stream);
/* head->seq reshard (inverse): x_head [B,S,h,D] -> x [B,S/P,H,D]. */
spa_status spa_reshard_head_to_seq(spa_plan *plan, const void *x_head, void *x, void *ws, void *stream);
spa_status spa_reshard_seq_to_head_local(spa_plan *plan, const void *const x[], void *const x_head[], void *ws,
                                         void *stream);
spa_status spa_reshard_head_to_seq_local(spa_plan *plan, const void *const x_head[], void *const x[], void *ws,
                                         void *stream);

/* Single-GPU attention kernel (tcgen05/TMEM/TMA), Alg. 1 line 3 for a group of heads:
 *   o[b, s, j, :] = softmax_t(q[b,s,j,:] . k[b,t,j,:] / sqrt(D)) v[b,t,j,:]
 * for b < B, s < Sq, j < n_heads, t < Skv.  Element (b, s, j, d) of q lives at
 * q + b*q_batch_stride + s*q_tok_stride + j*D + d (strides in elements, multiples of 8);
 * same for k, v (kv strides) and o (o strides).  D in {64, 96, 128}. */
spa_status spa_attention_fwd(const void *q, const void *k, const void *v, void *o, int B, int Sq, int Skv,
                             int n_heads, int D, long long q_tok_stride, long long q_batch_stride,
                             long long kv_tok_stride, long long kv_batch_stride, long long o_tok_stride,
                             long long o_batch_stride, void *stream);
/* The same with a key-padding mask: kv_len = device int32 [B] (NULL = none); keys t >= kv_len[b]
 * (clamped to [0, Skv]) take no part; kv_len[b] == 0 gives rows of 0 (R20). */
spa_status spa_attention_fwd_masked(const void *q, const void *k, const void *v, void *o, int B, int Sq, int Skv,
                                    int n_heads, int D, long long q_tok_stride, long long q_batch_stride,
                                    long long kv_tok_stride, long long kv_batch_stride, long long o_tok_stride,
                                    long long o_batch_stride, const int32_t *kv_len, void *stream);

/* The same kernel with the diagnostic outputs of SURVEY §8(c) c11: out_fp32 = 1 writes o as fp32 (the normalised
 * fp32 accumulator, element strides unchanged; bf16(o_fp32) equals the bf16 output bit for bit), and lse (NULL or
 * fp32 [B][Sq][n_heads]) receives each row's log-sum-exp ln sum_t exp(q.k_t / sqrt(D)) over its valid keys (-inf
 * when none) -- what partial results over disjoint key blocks are merged with (R21). */
spa_status spa_attention_fwd_ex(const void *q, const void *k, const void *v, void *o, int B, int Sq, int Skv,
                                int n_heads, int D, long long q_tok_stride, long long q_batch_stride,
                                long long kv_tok_stride, long long kv_batch_stride, long long o_tok_stride,
                                long long o_batch_stride, const int32_t *kv_len, int out_fp32, float *lse,
                                void *stream);

/* ------------------------------------------------------------------ host-side description (no GPU needed)
 * Buffers: 0 q, 1 k, 2 v, 3 out (the caller's, of source rank `src`), 4 ws (of rank `rank`). */
typedef struct {
    int src_buf, dst_buf;           /* buffer ids above */
    int src_rank, dst_rank;         /* whose buffer (for ws / user buffers) */
    long long src_off, dst_off;     /* byte offsets */
    long long count[4];             /* run index extents, outermost first */
    long long src_stride[4], dst_stride[4]; /* byte strides per level */
    long long run_bytes;            /* contiguous bytes per run (multiple of 64) */
} spa_copy_desc;
/* Messages of one stage's exchange as seen by `rank` (dir 0 = input Q/K/V, 1 = output O):
 * peer, direction (0 send, 1 recv), buffer id (4 = this rank's ws), byte offset, bytes.
 * For every ordered pair (p, q), p's sends to q and q's receives from p appear in the same
 * order, which is how they are matched (NCCL semantics). */
typedef struct {
    int peer, is_recv, buf;
    long long off, bytes;
} spa_msg;
spa_status spa_plan_describe_pack(const spa_plan *plan, int rank, spa_copy_desc *out, int max, int *n);
spa_status spa_plan_describe_unpack(const spa_plan *plan, int rank, spa_copy_desc *out, int max, int *n);
spa_status spa_plan_describe_messages(const spa_plan *plan, int stage, int dir, int rank, spa_msg *out, int max,
                                      int *n);
/* Ring plans: the NCCL messages of ring step t (0 <= t < nranks-1) as `rank` issues them: send K, send V to rank+1
 * (buf 1/2 = the caller's k/v at t = 0, else 4 = its ws receive slot (t-1)&1), receive K, V from rank-1 into ws slot
 * t&1.  USP plans: the step of the ring sub-plan, peers as global ranks. */
spa_status spa_plan_describe_ring(const spa_plan *plan, int step, int rank, spa_msg *out, int max, int *n);
/* Attention problem of stage k on owner rank `rank`: ws byte offsets of Q, K, V, O and Sq, Skv, n_heads. */
typedef struct {
    long long q_off, k_off, v_off, o_off;
    int B, Sq, Skv, n_heads;
    long long q_tok_stride, q_batch_stride, kv_tok_stride, kv_batch_stride; /* elements */
} spa_attn_desc;
spa_status spa_plan_describe_attention(const spa_plan *plan, int stage, int rank, spa_attn_desc *out);

/* ------------------------------------------------------------------ misc */
/* pad_heads: smallest multiple of n >= H; *pad_count = that - H. */
int spa_pad_heads(int H, int n, int *pad_count);
const char *spa_status_string(spa_status s);
const char *spa_last_error(void);
/* Library version string. */
const char *spa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPA_H_ */
