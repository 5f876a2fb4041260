// spa_api.cpp -- rank groups, plans, the per-stage pipeline scheduler and the C ABI (include/spa.h).
//
// Path of one call on one rank (Alg. 1, lines 1-13):
//   caller stream Sc: pack (seq->head send layout, all stages, one launch)
//   comm stream   Sm: in(0), in(1), out(0), in(2), out(1), ..., out(N-1)     (fixed issue order)
//   Sc:               attn(0), attn(1), ..., attn(N-1), unpack(+Psi_g)
//   events: pack -> in(0); in(k) -> attn(k); attn(k) -> out(k); out(N-1) -> unpack.
// in(k+1) and out(k-1) therefore overlap attn(k) (the paper's "record event / wait on CUDA
// stream / All_to_All", extended to the input side, R8).
// N_st = 1 is Ulysses.  Stage k = (head group kh, query chunk c), k = kh*C + c.
#include "../../include/spa.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <nvtx3/nvToolsExtCudaRt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "spa_internal.h"

using namespace spa;

namespace {

thread_local std::string g_last_error;

spa_status fail(spa_status s, const std::string &msg) {
    g_last_error = msg;
    return s;
}
#define SPA_CHECK_CUDA(expr)                                                                                   \
    do {                                                                                                       \
        cudaError_t _e = (expr);                                                                               \
        if (_e != cudaSuccess)                                                                                 \
            return fail(SPA_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));                   \
    } while (0)
#define SPA_CHECK_NCCL(expr)                                                                                   \
    do {                                                                                                       \
        ncclResult_t _r = (expr);                                                                              \
        if (_r != ncclSuccess) return fail(SPA_ERR_COMM, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
    } while (0)
#define SPA_TRY(expr)                       \
    do {                                    \
        spa_status _s = (expr);             \
        if (_s != SPA_OK) return _s;        \
    } while (0)

enum Kind { KIND_NCCL = 0, KIND_LOOPBACK = 1, KIND_HOST = 2, KIND_P2P = 3 };
enum Buf { BUF_Q = 0, BUF_K = 1, BUF_V = 2, BUF_OUT = 3, BUF_WS = 4, BUF_XHEAD = 5 };

long long align_up(long long x, long long a) { return (x + a - 1) / a * a; }

// NVTX range around the host-side enqueue of a call / step (tracing): visible in Nsight Systems next to
// the kernels and copies it issues; free when no tool is attached (NVTX3 is header-only, loaded on demand).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
    ~NvtxRange() { nvtxRangePop(); }
};

}  // namespace

struct spa_comm {
    int kind = KIND_HOST;
    int nranks = 1;
    int rank = 0;  // -1 for loopback
    int device = 0;
    ncclComm_t nccl = nullptr;
    cudaStream_t stream = nullptr;  // comm stream (highest priority), created on first use
};

namespace {

struct Split {
    int G_h, C, g;
    int n() const { return G_h * C; }
};

struct Ptrs {  // user buffers per source rank (loopback: arrays; NCCL: one entry)
    std::vector<const void *> q, k, v;
    std::vector<void *> out;
    std::vector<void *> xhead;  // reshard targets/sources per rank
    uint8_t *ws = nullptr;
};

}  // namespace

struct spa_plan {
    spa_comm *comm = nullptr;
    spa_shape sh{};
    int P = 1;      // ranks owning heads (all ranks)
    int Psrc = 1;   // ranks holding sequence shards
    int h = 1, S_l = 1;   // S_l: the longest sequence shard (buffer sizing)
    // source rank r holds tokens [start[r], start[r] + len[r]); lengths differ by <= 1 (R9), the first S % Psrc
    // ranks hold one token more
    std::vector<int> len, start;
    int Hp = 1;     // heads after padding to a multiple of P (== sh.H unless shape.pad_heads)
    const int32_t *kv_len = nullptr;   // key-padding lengths, device int32 [B] (spa_plan_set_kv_len) or NULL
    // ring plans (shape.ring = 1; R21): per-rank workspace = 2 K/V receive slots + P fp32 partials + lse
    bool ring = false;
    long long E_loc = 0;                         // B * S_l * H * D
    // USP hybrid (shape.ring = 1, shape.ulysses = U > 1): Ulysses over groups of U consecutive ranks, Ring over
    // the R = P/U groups.  Sub-comms / sub-plans owned by this plan; ws = 4 head-sharded tensors + sub-plan ws.
    int U = 1, R = 1;
    spa_comm *uly_comm = nullptr, *ring_comm = nullptr;
    spa_plan *uly_plan = nullptr, *ring_plan = nullptr;
    long long ws_total = -1;                     // >= 0: spa_plan_workspace_bytes returns this
    long long off_kvbuf = 0, off_parts = 0, off_lse = 0;
    long long off_ring_ws = -1;   // USP over P2P: the ring sub-plan's own workspace (the Ulysses one is at off_parts)
    Split split;
    // per-rank workspace layout (bytes)
    long long E_src = 0, E_own = 0;  // elements of one send-side / owner-side tensor
    long long off_sendQ = 0, off_sendK = 0, off_sendV = 0, off_orecv = 0;
    long long off_recvQ = 0, off_recvK = 0, off_recvV = 0, off_O = 0;
    long long ws_rank_bytes = 0;
    // options
    bool profile = false, skip_comm = false, coproc_busy = false, direct = false;
    int comm_sms = 0;   // SMs the persistent QKV GEMM leaves free for communication kernels (SPA_OPT_COMM_SMS)
    // measurement modes of loopback plans: only this virtual rank's launches and messages (SPA_OPT_RANK_ONLY, -1 =
    // all ranks); exchange messages as copy-engine cudaMemcpyAsync instead of the copy kernel (SPA_OPT_LOOPBACK_CE)
    int rank_only = -1;
    bool loopback_ce = false;
    // runtime resources (lazy)
    std::vector<cudaEvent_t> sync_ev;  // scheduling events (no timing)
    std::vector<cudaEvent_t> prof_ev;  // timing events
    spa_profile last{};
    bool have_profile = false;
    int prof_stages = 0;   // stages the last profiled call executed (spa_profile.n_stages)
    std::map<std::string, int> prof_idx;
    // P2P plans (KIND_P2P): every rank's workspace mapped into this process with CUDA IPC; per-call epoch
    // flags in each workspace's tail order the cross-process exchange (ready[src], in[k][src], out[k][src], uint32)
    std::vector<uint8_t *> peer_ws;   // [P]; own entry = the registered local workspace
    std::vector<void *> ipc_bases;    // opened peer allocations (closed by spa_plan_destroy)
    // NCCL plans with a registered symmetric window (spa_plan_window_register): peer_ws from NCCL's LSA mapping, and
    // the same peer-memory execution as P2P plans (copy engines / direct stores + epoch flags)
    ncclWindow_t win = nullptr;
    uint32_t epoch = 0;
    long long off_flags = 0, off_outbuf = 0;
    int n_flag_stages = 1;
    bool p2p_flush = false;
    int attn_launches = 0, copy_launches = 0, gemm_launches = 0;
    cudaStream_t sc_alt = nullptr;  // second compute stream: odd stages, so stage k+1 fills stage k's wave tail
    // stage window W (SPA_OPT_STAGE_WINDOW): up to W stages' attention in flight on W compute streams (the caller's, sc_alt,
    // then extra_streams); the comm stream issues in(0..W-1) up front and in(k+W) after out(k)
    int stage_window = 4;   // measured (profiles/r02/stage_window): flat at 720p, up to 1.8x at OSP with 24 stages
    std::vector<cudaStream_t> extra_streams;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;   // host-buffer SP calls: input / output copy streams
};

namespace spa {
cudaError_t nccl_window_bases(ncclWindow_t w, int n, uint8_t **bases, cudaStream_t st);   // nccl_window.cu
cudaError_t nccl_window_fill_pattern(uint32_t *lsa_self, long long n_words, uint32_t seed, cudaStream_t st);
ncclResult_t nccl_lsa_team(ncclComm_t comm, int *lsa_size, int *lsa_rank);
}  // namespace spa
namespace {

// ------------------------------------------------------------------ stage split (R7)
Split make_split(int h, int S_l, int stages) {
    Split s;
    s.G_h = std::gcd(stages, h);
    s.C = stages / s.G_h;
    s.g = h / s.G_h;
    return s;
}

bool is_source(const spa_plan *p, int r) { return r >= 0 && r < p->Psrc; }

// ------------------------------------------------------------------ offsets (elements)
// Query chunk c of source src covers its local tokens [clo(src, c), clo(src, c+1)) (R7; extents differ by <= 1).
long long clo(const spa_plan *p, const Split &s, int src, int c) { return (long long)c * p->len[src] / s.C; }
long long Lsrc(const spa_plan *p, const Split &s, int src, int c) { return clo(p, s, src, c + 1) - clo(p, s, src, c); }
// rows of stage chunk c on an owner (all sources' pieces) and the rows of all chunks before c
long long Lstage(const spa_plan *p, const Split &s, int c) {
    long long n = 0;
    for (int src = 0; src < p->Psrc; ++src) n += Lsrc(p, s, src, c);
    return n;
}
long long stage_prefix(const spa_plan *p, const Split &s, int c) {
    long long n = 0;
    for (int src = 0; src < p->Psrc; ++src) n += clo(p, s, src, c);
    return n;
}
long long src_prefix(const spa_plan *p, const Split &s, int c, int src) {
    long long n = 0;
    for (int q = 0; q < src; ++q) n += Lsrc(p, s, q, c);
    return n;
}
// send / orecv (source rank r): [kh][q][b][t][jj][d], q < P, t < len[r]
long long idx_send(const spa_plan *p, const Split &s, int r, int kh, int q, int b, long long t) {
    return ((((long long)kh * p->P + q) * p->sh.B + b) * p->len[r] + t) * s.g * p->sh.D;
}
// recvQ / O (owner side), stage (kh, c): [b][Lstage(c)][jj][d] at base(kh,c); source src's rows at src_prefix
long long base_stage(const spa_plan *p, const Split &s, int kh, int c) {
    return ((long long)kh * p->sh.B * p->sh.S + (long long)p->sh.B * stage_prefix(p, s, c)) * s.g * p->sh.D;
}
long long idx_qo(const spa_plan *p, const Split &s, int kh, int c, int b, int src) {
    return base_stage(p, s, kh, c) + ((long long)b * Lstage(p, s, c) + src_prefix(p, s, c, src)) * s.g * p->sh.D;
}
// recvK / recvV (owner side): [kh][b][S][jj][d]
long long idx_kv(const spa_plan *p, const Split &s, int kh, int b, int src) {
    return (((long long)kh * p->sh.B + b) * p->sh.S + p->start[src]) * s.g * p->sh.D;
}

struct Msg {
    int peer, is_recv, buf;
    long long off, bytes;
};

// Input exchange of stage k as seen by rank r (sends first, then receives).
// tensors: bitmask 1=Q 2=K 4=V.  q_recv_buf: BUF_WS (recvQ region) or BUF_XHEAD (reshard target).
void gen_in_msgs(const spa_plan *p, const Split &s, int k, int r, int tensors, int q_recv_buf, std::vector<Msg> &m) {
    const int kh = k / s.C, c = k % s.C;
    const long long run = (long long)s.g * p->sh.D * 2;
    const bool kv = (c == 0);
    if (is_source(p, r)) {
        const long long L = Lsrc(p, s, r, c), c0 = clo(p, s, r, c), n = p->len[r];
        for (int q = 0; q < p->P; ++q)
            for (int b = 0; b < p->sh.B; ++b) {
                if (tensors & 1) m.push_back({q, 0, BUF_WS, p->off_sendQ + idx_send(p, s, r, kh, q, b, c0) * 2, L * run});
                if (kv && (tensors & 2)) m.push_back({q, 0, BUF_WS, p->off_sendK + idx_send(p, s, r, kh, q, b, 0) * 2, n * run});
                if (kv && (tensors & 4)) m.push_back({q, 0, BUF_WS, p->off_sendV + idx_send(p, s, r, kh, q, b, 0) * 2, n * run});
            }
    }
    for (int src = 0; src < p->Psrc; ++src)
        for (int b = 0; b < p->sh.B; ++b) {
            const long long L = Lsrc(p, s, src, c), n = p->len[src];
            if (tensors & 1) {
                const long long rel = idx_qo(p, s, kh, c, b, src) * 2;
                m.push_back({src, 1, q_recv_buf, (q_recv_buf == BUF_WS ? p->off_recvQ : 0) + rel, L * run});
            }
            if (kv && (tensors & 2)) m.push_back({src, 1, BUF_WS, p->off_recvK + idx_kv(p, s, kh, b, src) * 2, n * run});
            if (kv && (tensors & 4)) m.push_back({src, 1, BUF_WS, p->off_recvV + idx_kv(p, s, kh, b, src) * 2, n * run});
        }
}

// Output exchange of stage k as seen by rank r.  o_send_buf: BUF_WS (O region) or BUF_XHEAD.
void gen_out_msgs(const spa_plan *p, const Split &s, int k, int r, int o_send_buf, std::vector<Msg> &m) {
    const int kh = k / s.C, c = k % s.C;
    const long long run = (long long)s.g * p->sh.D * 2;
    for (int src = 0; src < p->Psrc; ++src)
        for (int b = 0; b < p->sh.B; ++b) {
            const long long rel = idx_qo(p, s, kh, c, b, src) * 2;
            m.push_back({src, 0, o_send_buf, (o_send_buf == BUF_WS ? p->off_O : 0) + rel, Lsrc(p, s, src, c) * run});
        }
    if (is_source(p, r)) {
        const long long L = Lsrc(p, s, r, c), c0 = clo(p, s, r, c);
        for (int q = 0; q < p->P; ++q)
            for (int b = 0; b < p->sh.B; ++b)
                m.push_back({q, 1, BUF_WS, p->off_orecv + idx_send(p, s, r, kh, q, b, c0) * 2, L * run});
    }
}

// Real (unpadded) heads of head group kh owned by rank q: global heads q*h + kh*g + jj < H.
int real_heads(const spa_plan *p, const Split &s, int q, int kh) {
    return std::max(0, std::min(s.g, p->sh.H - (q * p->h + kh * s.g)));
}

// Pack (source rank): send[kh][q][b][t][jj][d] = X[b][t][q*h + kh*g + jj][d].
// One 4-level job when every head group is complete; with padded heads one job per (kh, q) that copies only
// the real heads of the group (pad-head slots of the send buffer are never written nor read as results).
void pack_jobs(const spa_plan *p, const Split &s, int r, const void *x, long long dst_off, uint8_t *ws,
               std::vector<CopyJob> &out, int kh_only = -1) {
    const long long D2 = (long long)p->sh.D * 2, H = p->sh.H, n = p->len[r];   // source rank r: n tokens
    const long long run = s.g * D2;
    // x == NULL / ws == NULL (describe): the job pointers hold plain byte offsets
    const uintptr_t xb = reinterpret_cast<uintptr_t>(x);
    const uintptr_t wb = ws ? reinterpret_cast<uintptr_t>(ws) + (uintptr_t)dst_off : 0;
    auto at = [](uintptr_t base, long long off) { return reinterpret_cast<uint8_t *>(base + (uintptr_t)off); };
    if (p->Hp == p->sh.H) {
        CopyJob j{};
        const int kh0 = kh_only < 0 ? 0 : kh_only;   // one head group only: its heads' runs for every destination
        j.src = at(xb, kh0 * s.g * D2);
        j.dst = at(wb, idx_send(p, s, r, kh0, 0, 0, 0) * 2);
        j.count[0] = kh_only < 0 ? s.G_h : 1; j.count[1] = p->P; j.count[2] = p->sh.B; j.count[3] = n;
        j.src_stride[0] = s.g * D2; j.src_stride[1] = p->h * D2; j.src_stride[2] = n * H * D2;
        j.src_stride[3] = H * D2;
        j.dst_stride[3] = run; j.dst_stride[2] = n * run; j.dst_stride[1] = p->sh.B * n * run;
        j.dst_stride[0] = p->P * p->sh.B * n * run;
        j.run_bytes = run;
        out.push_back(j);
        return;
    }
    for (int kh = 0; kh < s.G_h; ++kh)
        for (int q = 0; q < p->P; ++q) {
            const int nreal = real_heads(p, s, q, kh);
            if (nreal == 0 || (kh_only >= 0 && kh != kh_only)) continue;
            CopyJob j{};
            j.src = at(xb, (q * p->h + kh * s.g) * D2);
            j.dst = at(wb, idx_send(p, s, r, kh, q, 0, 0) * 2);
            j.count[0] = 1; j.count[1] = 1; j.count[2] = p->sh.B; j.count[3] = n;
            j.src_stride[2] = n * H * D2; j.src_stride[3] = H * D2;
            j.dst_stride[2] = n * run; j.dst_stride[3] = run;
            j.run_bytes = nreal * D2;
            out.push_back(j);
        }
}
// Unpack (source rank), Psi_g fused: out[b][t][q*h + kh*g + jj][d] = orecv[kh][q][b][t][jj][d]  (a5)
void unpack_jobs(const spa_plan *p, const Split &s, int r, uint8_t *ws, long long src_off, void *outp,
                 std::vector<CopyJob> &out, int kh_only = -1) {
    const size_t first = out.size();
    pack_jobs(p, s, r, nullptr, 0, nullptr, out, kh_only);
    for (size_t i = first; i < out.size(); ++i) {
        CopyJob &j = out[i];
        std::swap(j.src_stride, j.dst_stride);
        const uintptr_t src_rel = reinterpret_cast<uintptr_t>(j.dst), dst_rel = reinterpret_cast<uintptr_t>(j.src);
        j.src = reinterpret_cast<const uint8_t *>((ws ? reinterpret_cast<uintptr_t>(ws) + (uintptr_t)src_off : 0) + src_rel);
        j.dst = reinterpret_cast<uint8_t *>(reinterpret_cast<uintptr_t>(outp) + dst_rel);
    }
}

spa_copy_desc to_desc(const CopyJob &j, int sb, int sr, long long so, int db, int dr, long long dof) {
    spa_copy_desc d{};
    d.src_buf = sb; d.src_rank = sr; d.src_off = so; d.dst_buf = db; d.dst_rank = dr; d.dst_off = dof;
    for (int i = 0; i < 4; ++i) { d.count[i] = j.count[i]; d.src_stride[i] = j.src_stride[i]; d.dst_stride[i] = j.dst_stride[i]; }
    d.run_bytes = j.run_bytes;
    return d;
}

// ------------------------------------------------------------------ runtime helpers
spa_status ensure_stream(spa_comm *c) {
    if (c->stream) return SPA_OK;
    SPA_CHECK_CUDA(cudaSetDevice(c->device));
    int lo = 0, hi = 0;
    SPA_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SPA_CHECK_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi));
    nvtxNameCudaStreamA(c->stream, "spa comm stream");
    return SPA_OK;
}

spa_status ensure_events(spa_plan *p, size_t n_sync, size_t n_prof) {
    while (p->sync_ev.size() < n_sync) {
        cudaEvent_t e;
        SPA_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        p->sync_ev.push_back(e);
    }
    while (p->prof_ev.size() < n_prof) {
        cudaEvent_t e;
        SPA_CHECK_CUDA(cudaEventCreate(&e));
        p->prof_ev.push_back(e);
    }
    return SPA_OK;
}

struct Prof {  // named timing-event pairs recorded on a stream
    spa_plan *p;
    int next = 0;
    std::vector<std::pair<std::string, std::pair<int, int>>> spans;
    std::map<std::string, int> open;
    void begin(const std::string &name, cudaStream_t st) {
        if (!p->profile) return;
        int i = next++;
        cudaEventRecord(p->prof_ev[i], st);
        open[name] = i;
    }
    void end(const std::string &name, cudaStream_t st) {
        if (!p->profile) return;
        int i = next++;
        cudaEventRecord(p->prof_ev[i], st);
        spans.push_back({name, {open[name], i}});
    }
};

struct Exec {  // everything one call needs
    spa_plan *p;
    const Split *s;
    Ptrs ptr;
    cudaStream_t sc, sm, sc_alt;
    bool has_out = true;      // unpack at the end (false: reshard seq->head)
    bool has_attn = true;     // attention stage (false: reshard only)
    int in_tensors = 7;
    int q_recv_buf = BUF_WS, o_send_buf = BUF_WS;
    bool has_pack = true;
    // QKV projection fused with the pack: xin = hidden states [B, S_r, C] per local source rank
    bool qkv = false;
    std::vector<const void *> xin;
    const uint8_t *wp = nullptr;   // packed weight + bias (spa_plan_pack_qkv_weight)
    int C = 0;
    // host-buffer SP call: pinned host q/k/v/out per local source; ptr.q/k/v/out are then the device staging copies
    bool host = false;
    std::vector<const void *> hq, hk, hv;
    std::vector<void *> hout;
};

// ------------------------------------------------------------------ packed QKV weight
// [G_h][t < 3][q < P][r < g*D][C] bf16 = W[t*H*D + (q*h + kh*g)*D + r][C], then the bias in the same column order
// as fp32 [G_h][3][P][g*D] at a 256-byte aligned offset.  Head group kh's GEMM reads a contiguous [3*P*g*D][C].
long long qkv_cols(const spa_plan *p) { return 3LL * p->P * p->split.g * p->sh.D; }
long long qkv_bias_off(const spa_plan *p, int C) { return align_up((long long)p->split.G_h * qkv_cols(p) * C * 2, 256); }
long long qkv_packed_bytes(const spa_plan *p, int C) {
    return qkv_bias_off(p, C) + (long long)p->split.G_h * qkv_cols(p) * 4;
}

// GEMM of head group kh for the hidden states x of source rank r (M = B * len[r] tokens) into dst[t] + q*q_stride +
// m*row_stride + r (elements; see QkvProblem).
spa_status launch_qkv(spa_plan *p, const void *x, const uint8_t *wp, int C, int r, int kh, void *const dst[3],
                      long long q_stride, long long row_stride, cudaStream_t st) {
    QkvProblem g{};
    g.x = x;
    g.w = wp + (long long)kh * qkv_cols(p) * C * 2;
    g.bias = reinterpret_cast<const float *>(wp + qkv_bias_off(p, C)) + (long long)kh * qkv_cols(p);
    g.M = p->sh.B * p->len[r];
    g.N = (int)qkv_cols(p);
    g.K = C;
    for (int t = 0; t < 3; ++t) g.dst[t] = dst[t];
    g.q_stride = q_stride;
    g.row_stride = row_stride;
    g.cols_per_q = p->split.g * p->sh.D;
    g.cols_per_t = p->P * g.cols_per_q;
    g.reserve_sms = p->comm_sms;
    cudaError_t e = launch_qkv_gemm(g, st);
    if (e != cudaSuccess) return fail(SPA_ERR_CUDA, std::string("qkv gemm: ") + cudaGetErrorString(e));
    ++p->gemm_launches;
    return SPA_OK;
}

// Head group kh's projections of source rank r stored straight into every owner's receive regions (direct transport
// with the fused projections, one query chunk): peers[q] = owner q's workspace (local virtual rank or peer memory).
spa_status launch_qkv_direct(spa_plan *p, const Split &s, const void *x, const uint8_t *wp, int C, int r, int kh,
                             uint8_t *const peers[], cudaStream_t st) {
    if (p->P > kMaxDst) return fail(SPA_ERR_UNSUPPORTED, "direct projections: at most 16 owners");
    QkvProblem g{};
    g.x = x;
    g.w = wp + (long long)kh * qkv_cols(p) * C * 2;
    g.bias = reinterpret_cast<const float *>(wp + qkv_bias_off(p, C)) + (long long)kh * qkv_cols(p);
    g.M = p->sh.B * p->len[r];
    g.N = (int)qkv_cols(p);
    g.K = C;
    g.row_stride = (long long)s.g * p->sh.D;
    g.cols_per_q = s.g * p->sh.D;
    g.cols_per_t = p->P * g.cols_per_q;
    g.reserve_sms = p->comm_sms;
    for (int q = 0; q < p->P; ++q) g.peer[q] = peers[q];
    g.off[0] = p->off_recvQ / 2 + idx_qo(p, s, kh, 0, 0, r);   // [kh][c=0][b][S][g][D]: this source's rows
    g.off[1] = p->off_recvK / 2 + idx_kv(p, s, kh, 0, r);      // [kh][b][S][g][D]
    g.off[2] = p->off_recvV / 2 + idx_kv(p, s, kh, 0, r);
    g.rows_per_b = p->len[r];
    g.batch_rows = p->sh.S;
    if (s.C > kMaxQChunks) return fail(SPA_ERR_UNSUPPORTED, "direct projections: at most 32 query chunks");
    g.q_chunks = s.C;
    for (int c = 0; c < s.C; ++c) {   // chunk c of this source: stage (kh, c), after the earlier sources' pieces
        g.q_chunk_off[c] = p->off_recvQ / 2 + idx_qo(p, s, kh, c, 0, r);
        g.q_chunk_rows[c] = (int)Lstage(p, s, c);
    }
    cudaError_t e = launch_qkv_gemm(g, st);
    if (e != cudaSuccess) return fail(SPA_ERR_CUDA, std::string("qkv gemm (direct): ") + cudaGetErrorString(e));
    ++p->gemm_launches;
    return SPA_OK;
}

// The exchange runs on peer memory: CUDA-IPC (P2P) plans, and NCCL plans with a registered symmetric window.
bool peer_mem(const spa_plan *p) { return p->comm->kind == KIND_P2P || p->win != nullptr; }

uint8_t *resolve(const Exec &x, int rank, int buf, long long off) {
    const spa_plan *p = x.p;
    int idx = (p->comm->kind == KIND_LOOPBACK) ? rank : 0;
    switch (buf) {
        case BUF_WS:
            if (peer_mem(p)) return p->peer_ws[rank] + off;   // own or a peer's (CUDA IPC or NCCL window mapping)
            return x.ptr.ws + (p->comm->kind == KIND_LOOPBACK ? (long long)rank * p->ws_rank_bytes : 0) + off;
        case BUF_XHEAD: return reinterpret_cast<uint8_t *>(x.ptr.xhead[idx]) + off;
        case BUF_OUT: return reinterpret_cast<uint8_t *>(x.ptr.out[idx]) + off;
        case BUF_Q: return (uint8_t *)x.ptr.q[idx] + off;
        case BUF_K: return (uint8_t *)x.ptr.k[idx] + off;
        default: return (uint8_t *)x.ptr.v[idx] + off;
    }
}

// Compute stream of stage k: the caller's, sc_alt, then the plan's extra streams, round-robin over the stage window.
spa_status stage_stream(spa_plan *p, cudaStream_t sc, int k, cudaStream_t *out) {
    const int w = std::max(1, p->stage_window), i = k % w;
    if (i == 0) { *out = sc; return SPA_OK; }
    if (!p->sc_alt) SPA_CHECK_CUDA(cudaStreamCreateWithFlags(&p->sc_alt, cudaStreamNonBlocking));
    if (i == 1) { *out = p->sc_alt; return SPA_OK; }
    while ((int)p->extra_streams.size() < i - 1) {
        cudaStream_t st;
        SPA_CHECK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        p->extra_streams.push_back(st);
    }
    *out = p->extra_streams[i - 2];
    return SPA_OK;
}

// ------------------------------------------------------------------ P2P transport (CUDA IPC peer memory)
// Driver stream memory operations order the cross-process exchange without any kernel spinning: the sender's
// cuStreamWriteValue32 (with its implicit system-scope fence) stores the call's epoch into the receiver's flag
// after the data, the receiver's stream waits with cuStreamWaitValue32(>= epoch) before using it.
using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using AddrRangeFn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
struct Drv {
    WriteValue32Fn write32 = nullptr;
    WaitValue32Fn wait32 = nullptr;
    AddrRangeFn range = nullptr;
};
const Drv &drv() {
    static const Drv d = [] {
        Drv x;
        auto get = [](const char *name) -> void * {
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                return nullptr;
            return fn;
        };
        x.write32 = reinterpret_cast<WriteValue32Fn>(get("cuStreamWriteValue32"));
        x.wait32 = reinterpret_cast<WaitValue32Fn>(get("cuStreamWaitValue32"));
        x.range = reinterpret_cast<AddrRangeFn>(get("cuMemGetAddressRange"));
        return x;
    }();
    return d;
}
enum FlagKind { FLAG_READY = 0, FLAG_IN = 1, FLAG_OUT = 2 };
int flag_slot(const spa_plan *p, int kind, int k, int src) {
    return kind == FLAG_READY ? src : p->P + ((kind == FLAG_IN ? 0 : p->n_flag_stages) + k) * p->P + src;
}
long long flag_bytes(const spa_plan *p) { return 4LL * p->P * (1 + 2 * p->n_flag_stages); }
// this rank's flag `kind/k` in the flag block of every other rank := epoch
spa_status p2p_signal(spa_plan *p, cudaStream_t st, int kind, int k) {
    const int me = p->comm->rank;
    for (int q = 0; q < p->P; ++q) {
        if (q == me) continue;
        CUdeviceptr a = reinterpret_cast<CUdeviceptr>(p->peer_ws[q] + p->off_flags) + 4 * flag_slot(p, kind, k, me);
        if (drv().write32(reinterpret_cast<CUstream>(st), a, p->epoch, 0) != CUDA_SUCCESS)
            return fail(SPA_ERR_CUDA, "cuStreamWriteValue32 to a peer flag failed");
    }
    return SPA_OK;
}
// wait until every other rank's flag `kind/k` in this rank's flag block reached the epoch
spa_status p2p_wait(spa_plan *p, cudaStream_t st, int kind, int k) {
    const int me = p->comm->rank;
    for (int src = 0; src < p->P; ++src) {
        if (src == me) continue;
        CUdeviceptr a = reinterpret_cast<CUdeviceptr>(p->peer_ws[me] + p->off_flags) + 4 * flag_slot(p, kind, k, src);
        if (drv().wait32(reinterpret_cast<CUstream>(st), a, p->epoch,
                         CU_STREAM_WAIT_VALUE_GEQ | (p->p2p_flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0)) != CUDA_SUCCESS)
            return fail(SPA_ERR_CUDA, "cuStreamWaitValue32 on a flag failed");
    }
    return SPA_OK;
}
// single-peer forms (the ring): this rank's flag `kind/k` in rank dst's block; wait for src's flag in this rank's block
spa_status p2p_signal_one(spa_plan *p, cudaStream_t st, int kind, int k, int dst) {
    CUdeviceptr a = reinterpret_cast<CUdeviceptr>(p->peer_ws[dst] + p->off_flags) + 4 * flag_slot(p, kind, k, p->comm->rank);
    if (drv().write32(reinterpret_cast<CUstream>(st), a, p->epoch, 0) != CUDA_SUCCESS)
        return fail(SPA_ERR_CUDA, "cuStreamWriteValue32 to a peer flag failed");
    return SPA_OK;
}
spa_status p2p_wait_one(spa_plan *p, cudaStream_t st, int kind, int k, int src) {
    CUdeviceptr a = reinterpret_cast<CUdeviceptr>(p->peer_ws[p->comm->rank] + p->off_flags) + 4 * flag_slot(p, kind, k, src);
    if (drv().wait32(reinterpret_cast<CUstream>(st), a, p->epoch,
                     CU_STREAM_WAIT_VALUE_GEQ | (p->p2p_flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0)) != CUDA_SUCCESS)
        return fail(SPA_ERR_CUDA, "cuStreamWaitValue32 on a flag failed");
    return SPA_OK;
}
// every rank has finished its previous call (its buffers may be written): a cross-process barrier on `st`
spa_status p2p_barrier(spa_plan *p, cudaStream_t st) {
    SPA_TRY(p2p_signal(p, st, FLAG_READY, 0));
    return p2p_wait(p, st, FLAG_READY, 0);
}

template <class Gen>
spa_status match_and_copy(Exec &x, int me, Gen gen, cudaStream_t st) {
    // this rank's sends to q matched with q's receives from this rank, in order (NCCL semantics); copy-engine
    // copies straight into the peer's receive region (no SMs taken from the attention)
    spa_plan *p = x.p;
    std::vector<Msg> mine;
    gen(me, mine);
    for (int q = 0; q < p->P; ++q) {
        std::vector<Msg> theirs;
        gen(q, theirs);
        std::vector<const Msg *> sends, recvs;
        for (const Msg &g : mine) if (!g.is_recv && g.peer == q) sends.push_back(&g);
        for (const Msg &g : theirs) if (g.is_recv && g.peer == me) recvs.push_back(&g);
        if (sends.size() != recvs.size()) return fail(SPA_ERR_COMM, "p2p: unmatched messages");
        for (size_t i = 0; i < sends.size(); ++i) {
            if (sends[i]->bytes != recvs[i]->bytes) return fail(SPA_ERR_COMM, "p2p: size mismatch");
            SPA_CHECK_CUDA(cudaMemcpyAsync(resolve(x, q, recvs[i]->buf, recvs[i]->off),
                                           resolve(x, me, sends[i]->buf, sends[i]->off), (size_t)sends[i]->bytes,
                                           cudaMemcpyDeviceToDevice, st));
        }
    }
    return SPA_OK;
}

// Issue one stage exchange (dir 0 in, 1 out) on the comm stream.
spa_status run_exchange(Exec &x, int k, int dir) {
    spa_plan *p = x.p;
    if (p->skip_comm) return SPA_OK;
    if (peer_mem(p)) {
        auto gen = [&](int r, std::vector<Msg> &m) {
            if (dir == 0) gen_in_msgs(p, *x.s, k, r, x.in_tensors, x.q_recv_buf, m);
            else gen_out_msgs(p, *x.s, k, r, x.o_send_buf, m);
        };
        SPA_TRY(match_and_copy(x, p->comm->rank, gen, x.sm));
        return p2p_signal(p, x.sm, dir == 0 ? FLAG_IN : FLAG_OUT, k);
    }
    if (p->comm->kind == KIND_NCCL) {
        std::vector<Msg> m;
        if (dir == 0) gen_in_msgs(p, *x.s, k, p->comm->rank, x.in_tensors, x.q_recv_buf, m);
        else gen_out_msgs(p, *x.s, k, p->comm->rank, x.o_send_buf, m);
        SPA_CHECK_NCCL(ncclGroupStart());
        for (const Msg &g : m) {
            uint8_t *ptr = resolve(x, p->comm->rank, g.buf, g.off);
            if (g.is_recv) SPA_CHECK_NCCL(ncclRecv(ptr, (size_t)g.bytes, ncclUint8, g.peer, p->comm->nccl, x.sm));
            else SPA_CHECK_NCCL(ncclSend(ptr, (size_t)g.bytes, ncclUint8, g.peer, p->comm->nccl, x.sm));
        }
        SPA_CHECK_NCCL(ncclGroupEnd());
        return SPA_OK;
    }
    // loopback: match the i-th send p->q with the i-th receive of q from p (NCCL semantics) -> copies
    std::vector<std::vector<Msg>> per(p->P);
    for (int r = 0; r < p->P; ++r) {
        if (dir == 0) gen_in_msgs(p, *x.s, k, r, x.in_tensors, x.q_recv_buf, per[r]);
        else gen_out_msgs(p, *x.s, k, r, x.o_send_buf, per[r]);
    }
    std::vector<CopyJob> jobs;
    for (int src = 0; src < p->P; ++src)
        for (int dst = 0; dst < p->P; ++dst) {
            std::vector<const Msg *> sends, recvs;
            for (const Msg &g : per[src]) if (!g.is_recv && g.peer == dst) sends.push_back(&g);
            for (const Msg &g : per[dst]) if (g.is_recv && g.peer == src) recvs.push_back(&g);
            if (sends.size() != recvs.size()) return fail(SPA_ERR_COMM, "loopback: unmatched messages");
            if (p->rank_only >= 0 && src != p->rank_only && dst != p->rank_only) continue;
            for (size_t i = 0; i < sends.size(); ++i) {
                if (sends[i]->bytes != recvs[i]->bytes) return fail(SPA_ERR_COMM, "loopback: size mismatch");
                if (p->loopback_ce) {   // copy engines, as the P2P transport's staged exchange
                    SPA_CHECK_CUDA(cudaMemcpyAsync(resolve(x, dst, recvs[i]->buf, recvs[i]->off),
                                                   resolve(x, src, sends[i]->buf, sends[i]->off),
                                                   (size_t)sends[i]->bytes, cudaMemcpyDeviceToDevice, x.sm));
                    continue;
                }
                CopyJob j{};
                j.src = resolve(x, src, sends[i]->buf, sends[i]->off);
                j.dst = resolve(x, dst, recvs[i]->buf, recvs[i]->off);
                j.count[0] = j.count[1] = j.count[2] = j.count[3] = 1;
                j.run_bytes = sends[i]->bytes;
                jobs.push_back(j);
            }
        }
    if (!jobs.empty()) SPA_CHECK_CUDA(launch_copy_jobs(jobs.data(), (int)jobs.size(), x.sm, &p->copy_launches));
    return SPA_OK;
}

spa_status run_attention(Exec &x, int k, cudaStream_t st) {
    spa_plan *p = x.p;
    const Split &s = *x.s;
    const int kh = k / s.C, c = k % s.C;
    const long long Lst = Lstage(p, s, c);   // the stage's query rows (every source's chunk c)
    const int nr = (p->comm->kind == KIND_LOOPBACK) ? p->P : 1;
    for (int rr = 0; rr < nr; ++rr) {
        const int r = (p->comm->kind == KIND_LOOPBACK) ? rr : p->comm->rank;
        if (p->rank_only >= 0 && r != p->rank_only) continue;
        const int nreal = real_heads(p, s, r, kh);   // pad heads are not computed
        if (nreal == 0) continue;
        uint8_t *ws = resolve(x, r, BUF_WS, 0);
        AttnProblem a{};
        a.q = ws + p->off_recvQ + base_stage(p, s, kh, c) * 2;
        a.k = ws + p->off_recvK + idx_kv(p, s, kh, 0, 0) * 2;
        a.v = ws + p->off_recvV + idx_kv(p, s, kh, 0, 0) * 2;
        a.o = ws + p->off_O + base_stage(p, s, kh, c) * 2;
        a.B = p->sh.B; a.Sq = (int)Lst; a.Skv = p->sh.S; a.n_heads = nreal; a.D = p->sh.D;
        a.kv_len = p->kv_len;
        a.q_tok_stride = a.kv_tok_stride = a.o_tok_stride = (long long)s.g * p->sh.D;
        a.q_batch_stride = a.o_batch_stride = Lst * s.g * p->sh.D;
        a.kv_batch_stride = (long long)p->sh.S * s.g * p->sh.D;
        SPA_CHECK_CUDA(launch_attention(a, st));
        ++p->attn_launches;
    }
    return SPA_OK;
}

// QKV projections of every head group straight into the send layout (pack fused), one GEMM per (kh, local source);
// ev_gemm[kh] marks head group kh's send regions complete.
spa_status run_qkv_pack(Exec &x, cudaEvent_t *ev_gemm) {
    spa_plan *p = x.p;
    const Split &s = *x.s;
    const int nr = (p->comm->kind == KIND_LOOPBACK) ? p->Psrc : (is_source(p, p->comm->rank) ? 1 : 0);
    for (int kh = 0; kh < s.G_h; ++kh) {
        for (int i = 0; i < nr; ++i) {
            const int r = (p->comm->kind == KIND_LOOPBACK) ? i : p->comm->rank;
            if (p->rank_only >= 0 && r != p->rank_only) continue;
            uint8_t *ws = resolve(x, r, BUF_WS, 0);
            const long long base = idx_send(p, s, r, kh, 0, 0, 0) * 2;
            void *dst[3] = {ws + p->off_sendQ + base, ws + p->off_sendK + base, ws + p->off_sendV + base};
            SPA_TRY(launch_qkv(p, x.xin[i], x.wp, x.C, r, kh, dst, (long long)p->sh.B * p->len[r] * s.g * p->sh.D,
                               (long long)s.g * p->sh.D, x.sc));
        }
        SPA_CHECK_CUDA(cudaEventRecord(ev_gemm[kh], x.sc));
    }
    return SPA_OK;
}

// Host-buffer calls: the columns of head group kh's heads (for every destination rank) of one host [B, S_r, H, D]
// tensor, as 2-D copies (one per destination rank's head block); dir H2D or D2H.
spa_status copy_group_columns(const spa_plan *p, const Split &s, int r, int kh, void *dst, const void *src,
                              cudaMemcpyKind kind, cudaStream_t st) {
    const size_t row = (size_t)p->sh.H * p->sh.D * 2;
    for (int q = 0; q < p->P; ++q) {
        const int nreal = real_heads(p, s, q, kh);
        if (nreal == 0) continue;
        const size_t off = ((size_t)q * p->h + (size_t)kh * s.g) * p->sh.D * 2;
        SPA_CHECK_CUDA(cudaMemcpy2DAsync(reinterpret_cast<uint8_t *>(dst) + off, row,
                                         reinterpret_cast<const uint8_t *>(src) + off, row,
                                         (size_t)nreal * p->sh.D * 2, (size_t)p->sh.B * p->len[r], kind, st));
    }
    return SPA_OK;
}

// H2D of head group kh's Q/K/V columns on s_h2d, then its pack on the caller's stream; ev_ready[kh] = group kh's send
// regions complete (the input exchange of its first chunk waits for it)
spa_status run_host_pack(Exec &x, cudaEvent_t *ev_h2d, cudaEvent_t *ev_ready) {
    spa_plan *p = x.p;
    const Split &s = *x.s;
    const int nr = (p->comm->kind == KIND_LOOPBACK) ? p->Psrc : (is_source(p, p->comm->rank) ? 1 : 0);
    for (int kh = 0; kh < s.G_h; ++kh) {
        std::vector<CopyJob> jobs;
        for (int i = 0; i < nr; ++i) {
            const int r = (p->comm->kind == KIND_LOOPBACK) ? i : p->comm->rank;
            const void *hs[3] = {x.hq[i], x.hk[i], x.hv[i]};
            const void *ds[3] = {x.ptr.q[i], x.ptr.k[i], x.ptr.v[i]};
            for (int t = 0; t < 3; ++t)
                SPA_TRY(copy_group_columns(p, s, r, kh, const_cast<void *>(ds[t]), hs[t], cudaMemcpyHostToDevice,
                                           p->s_h2d));
            uint8_t *ws = resolve(x, r, BUF_WS, 0);
            pack_jobs(p, s, r, x.ptr.q[i], p->off_sendQ, ws, jobs, kh);
            pack_jobs(p, s, r, x.ptr.k[i], p->off_sendK, ws, jobs, kh);
            pack_jobs(p, s, r, x.ptr.v[i], p->off_sendV, ws, jobs, kh);
        }
        SPA_CHECK_CUDA(cudaEventRecord(ev_h2d[kh], p->s_h2d));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_h2d[kh], 0));
        if (!jobs.empty()) SPA_CHECK_CUDA(launch_copy_jobs(jobs.data(), (int)jobs.size(), x.sc, &p->copy_launches));
        SPA_CHECK_CUDA(cudaEventRecord(ev_ready[kh], x.sc));
    }
    return SPA_OK;
}

// Output of head group kh once its last stage's exchange is complete: unpack + Psi_g (copy kernel) and D2H of its
// columns, both on s_d2h (so neither waits behind later stages on the compute or comm streams)
spa_status run_host_unpack(Exec &x, int kh) {
    spa_plan *p = x.p;
    const Split &s = *x.s;
    const int nr = (p->comm->kind == KIND_LOOPBACK) ? p->Psrc : (is_source(p, p->comm->rank) ? 1 : 0);
    std::vector<CopyJob> jobs;
    for (int i = 0; i < nr; ++i) {
        const int r = (p->comm->kind == KIND_LOOPBACK) ? i : p->comm->rank;
        unpack_jobs(p, s, r, resolve(x, r, BUF_WS, 0), p->off_orecv, x.ptr.out[i], jobs, kh);
    }
    if (!jobs.empty()) SPA_CHECK_CUDA(launch_copy_jobs(jobs.data(), (int)jobs.size(), p->s_d2h, &p->copy_launches));
    for (int i = 0; i < nr; ++i) {
        const int r = (p->comm->kind == KIND_LOOPBACK) ? i : p->comm->rank;
        SPA_TRY(copy_group_columns(p, s, r, kh, x.hout[i], x.ptr.out[i], cudaMemcpyDeviceToHost, p->s_d2h));
    }
    return SPA_OK;
}

spa_status run_pack(Exec &x) {
    spa_plan *p = x.p;
    std::vector<CopyJob> jobs;
    const int nr = (p->comm->kind == KIND_LOOPBACK) ? p->Psrc : (is_source(p, p->comm->rank) ? 1 : 0);
    for (int i = 0; i < nr; ++i) {
        const int r = (p->comm->kind == KIND_LOOPBACK) ? i : p->comm->rank;
        if (p->rank_only >= 0 && r != p->rank_only) continue;
        uint8_t *ws = resolve(x, r, BUF_WS, 0);
        if (x.in_tensors & 1) pack_jobs(p, *x.s, r, x.ptr.q[i], p->off_sendQ, ws, jobs);
        if (x.in_tensors & 2) pack_jobs(p, *x.s, r, x.ptr.k[i], p->off_sendK, ws, jobs);
        if (x.in_tensors & 4) pack_jobs(p, *x.s, r, x.ptr.v[i], p->off_sendV, ws, jobs);
    }
    if (jobs.empty()) return SPA_OK;
    SPA_CHECK_CUDA(launch_copy_jobs(jobs.data(), (int)jobs.size(), x.sc, &p->copy_launches));
    return SPA_OK;
}

spa_status run_unpack(Exec &x) {
    spa_plan *p = x.p;
    std::vector<CopyJob> jobs;
    const int nr = (p->comm->kind == KIND_LOOPBACK) ? p->Psrc : (is_source(p, p->comm->rank) ? 1 : 0);
    for (int i = 0; i < nr; ++i) {
        const int r = (p->comm->kind == KIND_LOOPBACK) ? i : p->comm->rank;
        if (p->rank_only >= 0 && r != p->rank_only) continue;
        unpack_jobs(p, *x.s, r, resolve(x, r, BUF_WS, 0), p->off_orecv, x.ptr.out[i], jobs);
    }
    if (jobs.empty()) return SPA_OK;
    SPA_CHECK_CUDA(launch_copy_jobs(jobs.data(), (int)jobs.size(), x.sc, &p->copy_launches));
    return SPA_OK;
}

void finish_profile(spa_plan *p, const Prof &pr, int n_stages) {
    p->have_profile = false;
    if (!p->profile) return;
    p->prof_stages = n_stages;
    p->last = spa_profile{};
    p->last.n_stages = 0;
    p->prof_idx.clear();
    // stored as pairs; resolved on demand in spa_plan_last_profile (after the stream completes)
    p->prof_idx["__n"] = (int)pr.spans.size();
    int i = 0;
    for (auto &sp : pr.spans) {
        p->prof_idx[sp.first + "#b"] = sp.second.first;
        p->prof_idx[sp.first + "#e"] = sp.second.second;
        ++i;
    }
    p->have_profile = true;
}

// Direct transport (loopback model): every source's pack stores its runs straight into
// the owners' receive regions (no send staging, no exchange), and every stage's attention epilogue stores each
// output row straight into its source rank's [B, S_l, H, D] output at head k_orig (Psi_g and the output
// exchange fused: no orecv, no unpack).  On NVLink the same jobs / row tables use peer pointers of registered
// NCCL windows plus a per-stage barrier; on one GPU the "peers" are the virtual ranks' local buffers.
spa_status execute_direct(Exec &x) {
    NvtxRange range("spa: direct transport (loopback)");
    spa_plan *p = x.p;
    const Split &s = *x.s;
    const int N = s.n();
    const long long D2 = (long long)p->sh.D * 2, H = p->sh.H, run = s.g * D2;
    Prof pr{p};
    pr.begin("total", x.sc);
    pr.begin("pack", x.sc);
    std::vector<CopyJob> jobs;
    const long long offs[3] = {p->off_recvQ, p->off_recvK, p->off_recvV};
    if (x.qkv) {   // the fused projections store every owner's pieces themselves (projection + pack + exchange)
        std::vector<uint8_t *> peers(p->P);
        for (int q = 0; q < p->P; ++q) peers[q] = resolve(x, q, BUF_WS, 0);
        for (int kh = 0; kh < s.G_h; ++kh)
            for (int r = 0; r < p->Psrc; ++r) {
                if (p->rank_only >= 0 && r != p->rank_only) continue;
                SPA_TRY(launch_qkv_direct(p, s, x.xin[r], x.wp, x.C, r, kh, peers.data(), x.sc));
            }
    }
    for (int r = 0; r < p->Psrc && !x.qkv; ++r) {
        if (p->rank_only >= 0 && r != p->rank_only) continue;
        const void *xs[3] = {x.ptr.q[r], x.ptr.k[r], x.ptr.v[r]};
        const long long n = p->len[r];
        for (int t = 0; t < 3; ++t)
            for (int kh = 0; kh < s.G_h; ++kh)
                for (int q = 0; q < p->P; ++q) {
                    const int nreal = real_heads(p, s, q, kh);
                    if (nreal == 0) continue;
                    const uint8_t *src = reinterpret_cast<const uint8_t *>(xs[t]) + (q * p->h + kh * s.g) * D2;
                    uint8_t *wq = resolve(x, q, BUF_WS, offs[t]);
                    CopyJob j{};
                    j.count[0] = j.count[1] = 1;
                    j.count[2] = p->sh.B;
                    j.src_stride[2] = n * H * D2; j.src_stride[3] = H * D2;
                    j.dst_stride[3] = run;
                    j.run_bytes = nreal * D2;
                    if (t == 0) {   // Q: chunk c of this source's tokens -> stage (kh, c) of owner q
                        for (int c = 0; c < s.C; ++c) {
                            const long long L = Lsrc(p, s, r, c);
                            if (L == 0) continue;
                            CopyJob jc = j;
                            jc.src = src + clo(p, s, r, c) * H * D2;
                            jc.dst = wq + idx_qo(p, s, kh, c, 0, r) * 2;
                            jc.count[3] = L;
                            jc.dst_stride[2] = Lstage(p, s, c) * run;
                            jobs.push_back(jc);
                        }
                    } else {        // K / V: all of this source's tokens -> owner q's full-sequence region
                        j.src = src;
                        j.dst = wq + idx_kv(p, s, kh, 0, r) * 2;
                        j.count[3] = n;
                        j.dst_stride[2] = (long long)p->sh.S * run;
                        jobs.push_back(j);
                    }
                }
    }
    if (!jobs.empty()) SPA_CHECK_CUDA(launch_copy_jobs(jobs.data(), (int)jobs.size(), x.sc, &p->copy_launches));
    pr.end("pack", x.sc);
    // stages alternate between two streams so stage k+1 fills stage k's wave tail (as in execute())
    if (!p->sc_alt) SPA_CHECK_CUDA(cudaStreamCreateWithFlags(&p->sc_alt, cudaStreamNonBlocking));
    cudaEvent_t ev_pack = p->sync_ev[1], ev_alt = p->sync_ev[2];
    SPA_CHECK_CUDA(cudaEventRecord(ev_pack, x.sc));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(p->sc_alt, ev_pack, 0));
    for (int k = 0; k < N; ++k) {
        const int kh = k / s.C, c = k % s.C;
        const long long Lst = Lstage(p, s, c);
        const std::string an = "attn" + std::to_string(k);
        cudaStream_t st;
        SPA_TRY(stage_stream(p, x.sc, k, &st));
        if (st != x.sc && st != p->sc_alt) SPA_CHECK_CUDA(cudaStreamWaitEvent(st, ev_pack, 0));
        pr.begin(an, st);
        for (int r = 0; r < p->P; ++r) {   // owner r
            if (p->rank_only >= 0 && r != p->rank_only) continue;
            const int nreal = real_heads(p, s, r, kh);
            if (nreal == 0) continue;
            uint8_t *ws = resolve(x, r, BUF_WS, 0);
            AttnProblem a{};
            a.q = ws + p->off_recvQ + base_stage(p, s, kh, c) * 2;
            a.k = ws + p->off_recvK + idx_kv(p, s, kh, 0, 0) * 2;
            a.v = ws + p->off_recvV + idx_kv(p, s, kh, 0, 0) * 2;
            a.o = ws + p->off_O;   // unused (scattered output)
            a.B = p->sh.B; a.Sq = (int)Lst; a.Skv = p->sh.S; a.n_heads = nreal; a.D = p->sh.D;
            a.kv_len = p->kv_len;
            a.q_tok_stride = a.kv_tok_stride = (long long)s.g * p->sh.D;
            a.q_batch_stride = Lst * s.g * p->sh.D;
            a.kv_batch_stride = (long long)p->sh.S * s.g * p->sh.D;
            a.o_tok_stride = H * p->sh.D;
            a.o_batch_stride = 0;
            a.n_dst = p->Psrc;
            for (int q = 0; q < p->Psrc; ++q) {
                a.row_begin[q] = (int)src_prefix(p, s, c, q);
                a.dst[q] = reinterpret_cast<uint8_t *>(x.ptr.out[q]) +
                           ((clo(p, s, q, c) * H) + (long long)r * p->h + (long long)kh * s.g) * D2;
                a.dst_batch_stride[q] = (long long)p->len[q] * H * p->sh.D;
            }
            a.row_begin[p->Psrc] = (int)Lst;
            SPA_CHECK_CUDA(launch_attention(a, st));
            ++p->attn_launches;
        }
        pr.end(an, st);
    }
    SPA_CHECK_CUDA(cudaEventRecord(ev_alt, p->sc_alt));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_alt, 0));
    for (cudaStream_t st : p->extra_streams) {   // join the wider stage window (the event is reused in order)
        SPA_CHECK_CUDA(cudaEventRecord(ev_alt, st));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_alt, 0));
    }
    pr.end("total", x.sc);
    finish_profile(p, pr, N);
    return SPA_OK;
}

// Direct transport across processes (SURVEY f1 over NVLink / CUDA IPC): this rank's pack stores its runs straight
// into the owners' receive regions (peer pointers), its attention epilogues store every output row straight into the
// source rank's output landing buffer (ws region `outbuf`, [B, S_r, H, D], Psi_g fused), and each source copies its
// landing buffer to `out` once every owner signalled.  Same jobs / row tables as the loopback model above, with the
// peers' workspaces instead of local ones, and epoch flags instead of stream order.
spa_status execute_direct_p2p(Exec &x) {
    NvtxRange range("spa: direct transport (p2p)");
    spa_plan *p = x.p;
    const Split &s = *x.s;
    const int N = s.n(), me = p->comm->rank;
    const long long D2 = (long long)p->sh.D * 2, H = p->sh.H, run = s.g * D2;
    Prof pr{p};
    ++p->epoch;
    pr.begin("total", x.sc);
    SPA_TRY(p2p_barrier(p, x.sc));   // the pack below writes into the peers' receive regions
    pr.begin("pack", x.sc);
    std::vector<CopyJob> jobs;
    const long long offs[3] = {p->off_recvQ, p->off_recvK, p->off_recvV};
    // fused projections: head group kh's GEMM stores into every owner, then flags the group's stages
    std::vector<cudaEvent_t> ev_grp;
    if (x.qkv && is_source(p, me)) {
        std::vector<uint8_t *> peers(p->P);
        for (int q = 0; q < p->P; ++q) peers[q] = resolve(x, q, BUF_WS, 0);
        for (int kh = 0; kh < s.G_h; ++kh) {
            SPA_TRY(launch_qkv_direct(p, s, x.xin[0], x.wp, x.C, me, kh, peers.data(), x.sc));
            for (int c = 0; c < s.C && !p->skip_comm; ++c)   // every query chunk (stage) of head group kh
                SPA_TRY(p2p_signal(p, x.sc, FLAG_IN, kh * s.C + c));
            ev_grp.push_back(p->sync_ev[4 + kh]);
            SPA_CHECK_CUDA(cudaEventRecord(ev_grp.back(), x.sc));
        }
    }
    if (is_source(p, me) && !x.qkv) {
        const void *xs[3] = {x.ptr.q[0], x.ptr.k[0], x.ptr.v[0]};
        const long long n = p->len[me];
        for (int t = 0; t < 3; ++t)
            for (int kh = 0; kh < s.G_h; ++kh)
                for (int q = 0; q < p->P; ++q) {
                    const int nreal = real_heads(p, s, q, kh);
                    if (nreal == 0) continue;
                    const uint8_t *src = reinterpret_cast<const uint8_t *>(xs[t]) + (q * p->h + kh * s.g) * D2;
                    uint8_t *wq = resolve(x, q, BUF_WS, offs[t]);
                    CopyJob j{};
                    j.count[0] = j.count[1] = 1;
                    j.count[2] = p->sh.B;
                    j.src_stride[2] = n * H * D2; j.src_stride[3] = H * D2;
                    j.dst_stride[3] = run;
                    j.run_bytes = nreal * D2;
                    if (t == 0) {
                        for (int c = 0; c < s.C; ++c) {
                            const long long L = Lsrc(p, s, me, c);
                            if (L == 0) continue;
                            CopyJob jc = j;
                            jc.src = src + clo(p, s, me, c) * H * D2;
                            jc.dst = wq + idx_qo(p, s, kh, c, 0, me) * 2;
                            jc.count[3] = L;
                            jc.dst_stride[2] = Lstage(p, s, c) * run;
                            jobs.push_back(jc);
                        }
                    } else {
                        j.src = src;
                        j.dst = wq + idx_kv(p, s, kh, 0, me) * 2;
                        j.count[3] = n;
                        j.dst_stride[2] = (long long)p->sh.S * run;
                        jobs.push_back(j);
                    }
                }
    }
    if (!jobs.empty()) SPA_CHECK_CUDA(launch_copy_jobs(jobs.data(), (int)jobs.size(), x.sc, &p->copy_launches));
    pr.end("pack", x.sc);
    if (!p->skip_comm && !x.qkv) {
        SPA_TRY(p2p_signal(p, x.sc, FLAG_IN, 0));   // all of this rank's runs are in place (every stage)
        SPA_TRY(p2p_wait(p, x.sc, FLAG_IN, 0));
    }
    if (!p->sc_alt) SPA_CHECK_CUDA(cudaStreamCreateWithFlags(&p->sc_alt, cudaStreamNonBlocking));
    cudaEvent_t ev_pack = p->sync_ev[1], ev_alt = p->sync_ev[2];
    SPA_CHECK_CUDA(cudaEventRecord(ev_pack, x.sc));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(p->sc_alt, ev_pack, 0));
    for (int k = 0; k < N; ++k) {
        const int kh = k / s.C, c = k % s.C;
        const long long Lst = Lstage(p, s, c);
        const std::string an = "attn" + std::to_string(k);
        cudaStream_t st;
        SPA_TRY(stage_stream(p, x.sc, k, &st));
        if (st != x.sc && st != p->sc_alt) SPA_CHECK_CUDA(cudaStreamWaitEvent(st, ev_pack, 0));
        if (x.qkv) {   // this stage's pieces: the own GEMM's stores (head group kh) and every peer's flag for stage k
            if (kh < (int)ev_grp.size()) SPA_CHECK_CUDA(cudaStreamWaitEvent(st, ev_grp[kh], 0));
            if (!p->skip_comm) SPA_TRY(p2p_wait(p, st, FLAG_IN, k));
        }
        pr.begin(an, st);
        const int nreal = real_heads(p, s, me, kh);
        if (nreal > 0) {
            uint8_t *ws = resolve(x, me, BUF_WS, 0);
            AttnProblem a{};
            a.q = ws + p->off_recvQ + base_stage(p, s, kh, c) * 2;
            a.k = ws + p->off_recvK + idx_kv(p, s, kh, 0, 0) * 2;
            a.v = ws + p->off_recvV + idx_kv(p, s, kh, 0, 0) * 2;
            a.o = ws + p->off_O;
            a.B = p->sh.B; a.Sq = (int)Lst; a.Skv = p->sh.S; a.n_heads = nreal; a.D = p->sh.D;
            a.kv_len = p->kv_len;
            a.q_tok_stride = a.kv_tok_stride = (long long)s.g * p->sh.D;
            a.q_batch_stride = Lst * s.g * p->sh.D;
            a.kv_batch_stride = (long long)p->sh.S * s.g * p->sh.D;
            a.o_tok_stride = H * p->sh.D;
            a.o_batch_stride = 0;
            a.n_dst = p->Psrc;
            for (int q = 0; q < p->Psrc; ++q) {
                a.row_begin[q] = (int)src_prefix(p, s, c, q);
                a.dst[q] = resolve(x, q, BUF_WS, p->off_outbuf) +
                           ((clo(p, s, q, c) * H) + (long long)me * p->h + (long long)kh * s.g) * D2;
                a.dst_batch_stride[q] = (long long)p->len[q] * H * p->sh.D;
            }
            a.row_begin[p->Psrc] = (int)Lst;
            SPA_CHECK_CUDA(launch_attention(a, st));
            ++p->attn_launches;
        }
        pr.end(an, st);
    }
    SPA_CHECK_CUDA(cudaEventRecord(ev_alt, p->sc_alt));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_alt, 0));
    for (cudaStream_t st : p->extra_streams) {   // join the wider stage window (the event is reused in order)
        SPA_CHECK_CUDA(cudaEventRecord(ev_alt, st));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_alt, 0));
    }
    if (!p->skip_comm) {
        SPA_TRY(p2p_signal(p, x.sc, FLAG_OUT, 0));   // this owner's rows are in every source's landing buffer
        SPA_TRY(p2p_wait(p, x.sc, FLAG_OUT, 0));
    }
    if (is_source(p, me)) {
        pr.begin("unpack", x.sc);
        SPA_CHECK_CUDA(cudaMemcpyAsync(x.ptr.out[0], resolve(x, me, BUF_WS, p->off_outbuf),
                                       (size_t)p->sh.B * p->len[me] * H * D2, cudaMemcpyDeviceToDevice, x.sc));
        pr.end("unpack", x.sc);
    }
    pr.end("total", x.sc);
    finish_profile(p, pr, N);
    return SPA_OK;
}

// The whole call: single-rank fast path, else the staged pipeline.
spa_status execute(Exec &x) {
    NvtxRange range(x.qkv ? "spa: qkv + sp attention" : (x.has_attn ? "spa: sp attention" : "spa: reshard"));
    spa_plan *p = x.p;
    p->attn_launches = 0;
    p->copy_launches = 0;
    p->gemm_launches = 0;
    const Split &s = *x.s;
    const int N = s.n();
    SPA_TRY(ensure_events(p, 4 + 3 * (size_t)N + 3 * (size_t)s.G_h, p->profile ? 8 + 6 * (size_t)N : 0));
    // direct transport: the pack (or, with one query chunk, the fused projections) and the attention epilogue store to
    // the owners / sources themselves
    if (p->direct && p->P > 1 && x.has_attn && x.has_pack && x.has_out && !x.host && (!x.qkv || s.C <= kMaxQChunks))
        return peer_mem(p) ? execute_direct_p2p(x) : execute_direct(x);
    Prof pr{p};
    if (p->P == 1) {
        // one rank owns everything: attention straight on the caller's [B,S,H,D] buffers
        pr.begin("total", x.sc);
        if (x.has_attn) {
            AttnProblem a{};
            a.q = x.ptr.q[0]; a.k = x.ptr.k[0]; a.v = x.ptr.v[0]; a.o = x.ptr.out[0];
            if (x.qkv) {   // projections into the workspace's [B, S, H, D] Q, K, V (spa_plan_qkv_workspace_bytes)
                const long long E = (long long)p->sh.B * p->sh.S * p->sh.H * p->sh.D * 2;
                void *dst[3] = {x.ptr.ws, x.ptr.ws + E, x.ptr.ws + 2 * E};
                pr.begin("pack", x.sc);
                for (int kh = 0; kh < s.G_h; ++kh) {
                    void *d[3] = {(uint8_t *)dst[0] + (long long)kh * s.g * p->sh.D * 2,
                                  (uint8_t *)dst[1] + (long long)kh * s.g * p->sh.D * 2,
                                  (uint8_t *)dst[2] + (long long)kh * s.g * p->sh.D * 2};
                    SPA_TRY(launch_qkv(p, x.xin[0], x.wp, x.C, 0, kh, d, 0, (long long)p->sh.H * p->sh.D, x.sc));
                }
                pr.end("pack", x.sc);
                a.q = dst[0]; a.k = dst[1]; a.v = dst[2];
            }
            a.B = p->sh.B; a.Sq = a.Skv = p->sh.S; a.n_heads = p->sh.H; a.D = p->sh.D;
            a.kv_len = p->kv_len;
            a.q_tok_stride = a.kv_tok_stride = a.o_tok_stride = (long long)p->sh.H * p->sh.D;
            a.q_batch_stride = a.kv_batch_stride = a.o_batch_stride = (long long)p->sh.S * p->sh.H * p->sh.D;
            pr.begin("attn0", x.sc);
            SPA_CHECK_CUDA(launch_attention(a, x.sc));
            pr.end("attn0", x.sc);
            ++p->attn_launches;
        } else {
            const long long bytes = (long long)p->sh.B * p->sh.S * p->sh.H * p->sh.D * 2;
            const void *src = x.has_out ? x.ptr.xhead[0] : x.ptr.q[0];
            void *dst = x.has_out ? x.ptr.out[0] : x.ptr.xhead[0];
            SPA_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, x.sc));
        }
        pr.end("total", x.sc);
        finish_profile(p, pr, 1);
        return SPA_OK;
    }
    SPA_TRY(ensure_stream(p->comm));
    x.sm = p->comm->stream;
    if (!p->sc_alt) SPA_CHECK_CUDA(cudaStreamCreateWithFlags(&p->sc_alt, cudaStreamNonBlocking));
    x.sc_alt = p->sc_alt;
    cudaEvent_t *ev = p->sync_ev.data();
    cudaEvent_t ev_entry = ev[0], ev_pack = ev[1], ev_done = ev[2];
    cudaEvent_t *ev_in = ev + 4, *ev_attn = ev + 4 + N, *ev_out = ev + 4 + 2 * N, *ev_gemm = ev + 4 + 3 * N;
    cudaEvent_t *ev_h2d = ev_gemm + s.G_h, *ev_hout = ev_gemm + 2 * s.G_h;
    if (x.host) {
        if (!p->s_h2d) SPA_CHECK_CUDA(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking));
        if (!p->s_d2h) SPA_CHECK_CUDA(cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking));
        SPA_CHECK_CUDA(cudaEventRecord(ev_entry, x.sc));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(p->s_h2d, ev_entry, 0));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(p->s_d2h, ev_entry, 0));
    }

    pr.begin("total", x.sc);
    SPA_CHECK_CUDA(cudaEventRecord(ev_entry, x.sc));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sm, ev_entry, 0));
    const bool p2p = peer_mem(p);
    if (p2p) {   // a new epoch; no rank writes into a peer before that peer finished its previous call
        ++p->epoch;
        SPA_TRY(p2p_barrier(p, x.sm));
    }
    if (x.has_pack) {
        pr.begin("pack", x.sc);
        if (x.qkv) SPA_TRY(run_qkv_pack(x, ev_gemm));
        else if (x.host) SPA_TRY(run_host_pack(x, ev_h2d, ev_gemm));
        else SPA_TRY(run_pack(x));
        pr.end("pack", x.sc);
    }
    SPA_CHECK_CUDA(cudaEventRecord(ev_pack, x.sc));
    // the staged pack is one launch; the fused projections / host copies complete head group by head group (ev_gemm)
    const bool per_group = x.qkv || x.host;
    if (!per_group) SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sm, ev_pack, 0));

    auto issue_in = [&](int k) -> spa_status {
        NvtxRange r_in("spa: input exchange");
        if (per_group && k % s.C == 0) SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sm, ev_gemm[k / s.C], 0));
        const std::string nm = "in" + std::to_string(k);
        pr.begin(nm, x.sm);
        SPA_TRY(run_exchange(x, k, 0));
        pr.end(nm, x.sm);
        SPA_CHECK_CUDA(cudaEventRecord(ev_in[k], x.sm));
        return SPA_OK;
    };
    if (x.has_attn) {
        const int W = std::max(1, p->stage_window);
        for (int k = 0; k < std::min(W, N); ++k) SPA_TRY(issue_in(k));
        for (int k = 0; k < N; ++k) {
            cudaStream_t st;
            SPA_TRY(stage_stream(p, x.sc, k, &st));
            NvtxRange r_stage("spa: stage");
            SPA_CHECK_CUDA(cudaStreamWaitEvent(st, ev_in[k], 0));
            if (p2p && !p->skip_comm) SPA_TRY(p2p_wait(p, st, FLAG_IN, k));   // the peers' pieces of stage k
            const std::string an = "attn" + std::to_string(k);
            pr.begin(an, st);
            SPA_TRY(run_attention(x, k, st));
            pr.end(an, st);
            SPA_CHECK_CUDA(cudaEventRecord(ev_attn[k], st));
            SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sm, ev_attn[k], 0));
            const std::string on = "out" + std::to_string(k);
            pr.begin(on, x.sm);
            SPA_TRY(run_exchange(x, k, 1));
            pr.end(on, x.sm);
            SPA_CHECK_CUDA(cudaEventRecord(ev_out[k], x.sm));
            if (x.host && k % s.C == s.C - 1) {   // head group k / C complete: its output goes home now
                const int kh = k / s.C;
                SPA_CHECK_CUDA(cudaStreamWaitEvent(p->s_d2h, ev_out[k], 0));
                if (p2p && !p->skip_comm)
                    for (int kk = kh * s.C; kk <= k; ++kk) SPA_TRY(p2p_wait(p, p->s_d2h, FLAG_OUT, kk));
                SPA_TRY(run_host_unpack(x, kh));
                SPA_CHECK_CUDA(cudaEventRecord(ev_hout[kh], p->s_d2h));
            }
            if (k + W < N) SPA_TRY(issue_in(k + W));
        }
        SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_out[N - 1], 0));
        if (x.host) SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_hout[s.G_h - 1], 0));
        if (p2p && !p->skip_comm && !x.host)
            for (int k = 0; k < N; ++k) SPA_TRY(p2p_wait(p, x.sc, FLAG_OUT, k));   // every owner's output rows
    } else if (!x.has_out) {
        // reshard seq->head: the one input exchange only
        SPA_TRY(issue_in(0));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_in[0], 0));
        if (p2p) {   // the pieces landed in this rank's recvQ region ([B][S][h][D]): to the caller's x_head
            if (!p->skip_comm) SPA_TRY(p2p_wait(p, x.sc, FLAG_IN, 0));
            SPA_CHECK_CUDA(cudaMemcpyAsync(x.ptr.xhead[0], resolve(x, p->comm->rank, BUF_WS, p->off_recvQ),
                                           (size_t)p->E_own * 2, cudaMemcpyDeviceToDevice, x.sc));
        }
    } else {
        // reshard head->seq: the one output exchange only
        pr.begin("out0", x.sm);
        SPA_TRY(run_exchange(x, 0, 1));
        pr.end("out0", x.sm);
        SPA_CHECK_CUDA(cudaEventRecord(ev_out[0], x.sm));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_out[0], 0));
        if (p2p && !p->skip_comm) SPA_TRY(p2p_wait(p, x.sc, FLAG_OUT, 0));
    }
    if (x.has_out && !x.host) {
        pr.begin("unpack", x.sc);
        SPA_TRY(run_unpack(x));
        pr.end("unpack", x.sc);
    }
    pr.end("total", x.sc);
    // make the comm stream's tail visible to later work on the caller's stream
    SPA_CHECK_CUDA(cudaEventRecord(ev_done, x.sm));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(x.sc, ev_done, 0));
    finish_profile(p, pr, x.has_attn ? N : 1);
    return SPA_OK;
}

spa_status check_ptr(const void *ptr, const char *what) {
    if (!ptr) return fail(SPA_ERR_INVALID, std::string(what) + " is NULL");
    if (reinterpret_cast<uintptr_t>(ptr) % 16) return fail(SPA_ERR_INVALID, std::string(what) + " not 16-byte aligned");
    return SPA_OK;
}

spa_status prepare(spa_plan *p, Exec &x, void *ws, void *stream, bool local) {
    if (!p) return fail(SPA_ERR_INVALID, "plan is NULL");
    if (p->comm->kind == KIND_HOST) return fail(SPA_ERR_UNSUPPORTED, "host-only comm cannot execute");
    if (local != (p->comm->kind == KIND_LOOPBACK))
        return fail(SPA_ERR_INVALID, local ? "*_local calls need a loopback plan" : "loopback plans need the *_local calls");
    if (p->P > 1) SPA_TRY(check_ptr(ws, "ws"));
    if (p->comm->kind == KIND_P2P && p->P > 1) {
        if (p->peer_ws.empty()) return fail(SPA_ERR_INVALID, "p2p plan: call spa_plan_ipc_open first");
        if (ws != p->peer_ws[p->comm->rank]) return fail(SPA_ERR_INVALID, "p2p plan: ws is not the registered workspace");
    }
    if (p->win && ws != p->peer_ws[p->comm->rank])
        return fail(SPA_ERR_INVALID, "NCCL window plan: ws is not the registered window");
    if (p->comm->kind == KIND_NCCL && p->direct && !p->win && p->P > 1)
        return fail(SPA_ERR_INVALID, "direct transport on an NCCL plan: register the workspace (spa_plan_window_register)");
    x.p = p;
    x.ptr.ws = reinterpret_cast<uint8_t *>(ws);
    x.sc = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = cudaSetDevice(p->comm->device);
    if (e != cudaSuccess) return fail(SPA_ERR_CUDA, cudaGetErrorString(e));
    return SPA_OK;
}

spa_status attention_call(spa_plan *p, int nsrc_ptrs, const void *const q[], const void *const k[],
                          const void *const v[], void *const out[], void *ws, void *stream, bool local, bool ulysses) {
    if (p && p->ring) return fail(SPA_ERR_INVALID, "ring plan: use spa_ring_attention");
    Exec x{};
    SPA_TRY(prepare(p, x, ws, stream, local));
    Split one = make_split(p->h, p->S_l, 1);
    x.s = ulysses ? &one : &p->split;
    for (int i = 0; i < nsrc_ptrs; ++i) {
        SPA_TRY(check_ptr(q[i], "q")); SPA_TRY(check_ptr(k[i], "k"));
        SPA_TRY(check_ptr(v[i], "v")); SPA_TRY(check_ptr(out[i], "out"));
        x.ptr.q.push_back(q[i]); x.ptr.k.push_back(k[i]); x.ptr.v.push_back(v[i]); x.ptr.out.push_back(out[i]);
    }
    return execute(x);
}

int n_local_srcs(const spa_plan *p) { return p->comm->kind == KIND_LOOPBACK ? p->Psrc : 1; }

}  // namespace

// ------------------------------------------------------------------ USP hybrid plan (R21)
// Ranks p = rho*U + u: Ulysses group rho = ranks [rho*U, rho*U+U), ring index u.  Step 1: seq->head all-to-all
// inside each group (heads [u*H/U, (u+1)*H/U) of the group's U*S_l tokens on rank (rho, u)); step 2: Ring
// attention over the R groups among the ranks with the same u; step 3: head->seq all-to-all inside the group.
static spa_status create_usp_plan(spa_plan **plan, spa_comm *comm, const spa_shape &s) {
    const int P = comm->nranks, U = s.ulysses;
    if (P % U) return fail(SPA_ERR_SHAPE, "ulysses degree must divide nranks");
    if (s.H % U) return fail(SPA_ERR_SHAPE, "H must be divisible by the ulysses degree");
    if (s.S % P) return fail(SPA_ERR_SHAPE, "S must be divisible by nranks");
    if (s.n_src != 0 && s.n_src != P) return fail(SPA_ERR_SHAPE, "USP plans have no co-processor ranks");
    const int R = P / U;
    spa_plan *p = new spa_plan;
    p->comm = comm; p->sh = s; p->P = P; p->Psrc = P; p->ring = true; p->U = U; p->R = R;
    p->Hp = s.H; p->h = s.H; p->S_l = s.S / P;
    p->split = make_split(1, p->S_l, 1);
    p->E_loc = (long long)s.B * p->S_l * s.H * s.D;
    auto cleanup = [&](spa_status st) { spa_plan_destroy(p); return st; };
    spa_status st = SPA_OK;
    if (comm->kind == KIND_LOOPBACK) {
        st = spa_comm_init_loopback(&p->uly_comm, U, comm->device);
        if (st == SPA_OK) st = spa_comm_init_loopback(&p->ring_comm, R, comm->device);
    } else if (comm->kind == KIND_HOST) {
        st = spa_comm_init_host(&p->uly_comm, U, comm->rank % U);
        if (st == SPA_OK) st = spa_comm_init_host(&p->ring_comm, R, comm->rank / U);
    } else if (comm->kind == KIND_P2P) {   // sub-groups of the same processes; mapped by spa_plan_ipc_open
        st = spa_comm_init_p2p(&p->uly_comm, U, comm->rank % U, comm->device);
        if (st == SPA_OK) st = spa_comm_init_p2p(&p->ring_comm, R, comm->rank / U, comm->device);
    } else {
        st = spa_comm_split(comm, comm->rank / U, comm->rank % U, &p->uly_comm);
        if (st == SPA_OK) st = spa_comm_split(comm, comm->rank % U, comm->rank / U, &p->ring_comm);
    }
    if (st != SPA_OK) return cleanup(st);
    spa_shape us{s.B, U * p->S_l, s.H, s.D, 1, 0, 0, 0, 0};
    spa_shape rs{s.B, s.S, s.H / U, s.D, 1, 0, 0, 1, 0};
    st = spa_plan_create(&p->uly_plan, p->uly_comm, &us);
    if (st == SPA_OK) st = spa_plan_create(&p->ring_plan, p->ring_comm, &rs);
    if (st != SPA_OK) return cleanup(st);
    size_t wu = 0, wr = 0;
    spa_plan_workspace_bytes(p->uly_plan, &wu);
    spa_plan_workspace_bytes(p->ring_plan, &wr);
    const int nloc = comm->kind == KIND_LOOPBACK ? P : 1;
    p->off_kvbuf = 0;   // head-sharded Q, K, V, O per (local) rank: [nloc][4][E_loc] bf16
    p->off_parts = align_up((long long)nloc * 4 * p->E_loc * 2, 256);   // sub-plan workspace
    if (comm->kind == KIND_P2P) {   // separate regions: each sub-plan's epoch flags persist across calls
        p->off_ring_ws = align_up(p->off_parts + (long long)wu, 256);
        p->ws_total = p->off_ring_ws + (long long)wr;
    } else {
        p->ws_total = p->off_parts + (long long)std::max(wu, wr);
    }
    *plan = p;
    return SPA_OK;
}

static spa_status usp_call(spa_plan *p, const void *const q[], const void *const k[], const void *const v[],
                           void *const out[], void *ws, void *stream, bool local) {
    if (p->comm->kind == KIND_HOST) return fail(SPA_ERR_UNSUPPORTED, "host-only comm cannot execute");
    if (local != (p->comm->kind == KIND_LOOPBACK))
        return fail(SPA_ERR_INVALID, local ? "*_local calls need a loopback plan" : "loopback plans need the *_local calls");
    SPA_TRY(check_ptr(ws, "ws"));
    const int U = p->U, R = p->R, nloc = local ? p->P : 1;
    for (int i = 0; i < nloc; ++i) {
        SPA_TRY(check_ptr(q[i], "q")); SPA_TRY(check_ptr(k[i], "k"));
        SPA_TRY(check_ptr(v[i], "v")); SPA_TRY(check_ptr(out[i], "out"));
    }
    SPA_TRY(ensure_events(p, 0, p->profile ? 2 : 0));
    Prof pr{p};
    pr.begin("total", reinterpret_cast<cudaStream_t>(stream));
    auto done = [&]() {
        pr.end("total", reinterpret_cast<cudaStream_t>(stream));
        finish_profile(p, pr, 1);   // attn_ms[0] = the ring sub-plan's call (spa_plan_last_profile)
        return SPA_OK;
    };
    uint8_t *w = reinterpret_cast<uint8_t *>(ws);
    uint8_t *sub_ws = w + p->off_parts;
    uint8_t *ring_ws = p->off_ring_ws >= 0 ? w + p->off_ring_ws : sub_ws;
    auto head = [&](int i, int t) { return w + ((long long)i * 4 + t) * p->E_loc * 2; };   // t: 0 Q 1 K 2 V 3 O
    const void *const *in[3] = {q, k, v};
    if (!local) {
        for (int t = 0; t < 3; ++t) SPA_TRY(spa_reshard_seq_to_head(p->uly_plan, in[t][0], head(0, t), sub_ws, stream));
        SPA_TRY(spa_ring_attention(p->ring_plan, head(0, 0), head(0, 1), head(0, 2), head(0, 3), ring_ws, stream));
        SPA_TRY(spa_reshard_head_to_seq(p->uly_plan, head(0, 3), out[0], sub_ws, stream));
        return done();
    }
    std::vector<const void *> xs(U);
    std::vector<void *> hs(U);
    for (int rho = 0; rho < R; ++rho)   // step 1 per Ulysses group
        for (int t = 0; t < 3; ++t) {
            for (int u = 0; u < U; ++u) { xs[u] = in[t][rho * U + u]; hs[u] = head(rho * U + u, t); }
            SPA_TRY(spa_reshard_seq_to_head_local(p->uly_plan, xs.data(), hs.data(), sub_ws, stream));
        }
    std::vector<const void *> rq(R), rk(R), rv(R);
    std::vector<void *> ro(R);
    for (int u = 0; u < U; ++u) {   // step 2 per ring
        for (int rho = 0; rho < R; ++rho) {
            const int i = rho * U + u;
            rq[rho] = head(i, 0); rk[rho] = head(i, 1); rv[rho] = head(i, 2); ro[rho] = head(i, 3);
        }
        SPA_TRY(spa_ring_attention_local(p->ring_plan, rq.data(), rk.data(), rv.data(), ro.data(), sub_ws, stream));
    }
    std::vector<void *> os(U);
    for (int rho = 0; rho < R; ++rho) {   // step 3 per Ulysses group
        for (int u = 0; u < U; ++u) { hs[u] = head(rho * U + u, 3); os[u] = out[rho * U + u]; }
        std::vector<const void *> hc(hs.begin(), hs.end());
        SPA_TRY(spa_reshard_head_to_seq_local(p->uly_plan, hc.data(), os.data(), sub_ws, stream));
    }
    return done();
}

// ==================================================================== C ABI
extern "C" {

const char *spa_version(void) { return "spa 0.1 (sm_100a tcgen05)"; }

const char *spa_status_string(spa_status s) {
    switch (s) {
        case SPA_OK: return "SPA_OK";
        case SPA_ERR_INVALID: return "SPA_ERR_INVALID";
        case SPA_ERR_SHAPE: return "SPA_ERR_SHAPE";
        case SPA_ERR_UNSUPPORTED: return "SPA_ERR_UNSUPPORTED";
        case SPA_ERR_CUDA: return "SPA_ERR_CUDA";
        case SPA_ERR_COMM: return "SPA_ERR_COMM";
        case SPA_ERR_BUSY: return "SPA_ERR_BUSY";
    }
    return "SPA_ERR_UNKNOWN";
}

const char *spa_last_error(void) { return g_last_error.c_str(); }

int spa_pad_heads(int H, int n, int *pad_count) {
    if (H < 1 || n < 1) {
        if (pad_count) *pad_count = 0;
        return -1;
    }
    const int hp = (H + n - 1) / n * n;
    if (pad_count) *pad_count = hp - H;
    return hp;
}

spa_status spa_get_unique_id(uint8_t id[128]) {
    if (!id) return fail(SPA_ERR_INVALID, "id is NULL");
    ncclUniqueId u;
    SPA_CHECK_NCCL(ncclGetUniqueId(&u));
    static_assert(sizeof(u.internal) == 128, "nccl unique id size");
    memcpy(id, u.internal, 128);
    return SPA_OK;
}

spa_status spa_comm_init(spa_comm **comm, const uint8_t id[128], int nranks, int rank, int device) {
    return spa_comm_init_config(comm, id, nranks, rank, device, nullptr);
}

spa_status spa_comm_init_config(spa_comm **comm, const uint8_t id[128], int nranks, int rank, int device,
                                const spa_comm_config *cfg) {
    if (!comm || !id) return fail(SPA_ERR_INVALID, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SPA_ERR_INVALID, "bad rank/nranks");
    if (cfg && (cfg->min_ctas < 0 || cfg->max_ctas < 0 || (cfg->max_ctas && cfg->min_ctas > cfg->max_ctas)))
        return fail(SPA_ERR_INVALID, "bad CTA bounds");
    if (cfg && (cfg->cta_policy < 0 || cfg->cta_policy > 2)) return fail(SPA_ERR_INVALID, "bad CTA policy");
    SPA_CHECK_CUDA(cudaSetDevice(device));
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclComm_t nc;
    ncclConfig_t nccfg = NCCL_CONFIG_INITIALIZER;
    // SM budget of NCCL's kernels while the attention grid occupies the GPU (NCCL's own env variables,
    // e.g. NCCL_MAX_CTAS, still apply when a field is left at 0)
    if (cfg) {
        if (cfg->min_ctas) nccfg.minCTAs = cfg->min_ctas;
        if (cfg->max_ctas) nccfg.maxCTAs = cfg->max_ctas;
        if (cfg->cta_policy) nccfg.CTAPolicy = cfg->cta_policy;
    }
    SPA_CHECK_NCCL(ncclCommInitRankConfig(&nc, nranks, u, rank, &nccfg));
    spa_comm *c = new spa_comm;
    c->kind = KIND_NCCL; c->nranks = nranks; c->rank = rank; c->device = device; c->nccl = nc;
    *comm = c;
    return SPA_OK;
}

spa_status spa_comm_init_loopback(spa_comm **comm, int nvirtual, int device) {
    if (!comm || nvirtual < 1) return fail(SPA_ERR_INVALID, "bad loopback arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(SPA_ERR_CUDA, "no such CUDA device");
    spa_comm *c = new spa_comm;
    c->kind = KIND_LOOPBACK; c->nranks = nvirtual; c->rank = -1; c->device = device;
    *comm = c;
    return SPA_OK;
}

spa_status spa_comm_init_p2p(spa_comm **comm, int nranks, int rank, int device) {
    if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(SPA_ERR_INVALID, "bad p2p comm arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(SPA_ERR_CUDA, "no such CUDA device");
    if (!drv().write32 || !drv().wait32 || !drv().range)
        return fail(SPA_ERR_UNSUPPORTED, "driver lacks stream memory operations");
    spa_comm *c = new spa_comm;
    c->kind = KIND_P2P; c->nranks = nranks; c->rank = rank; c->device = device;
    *comm = c;
    return SPA_OK;
}

spa_status spa_plan_ipc_handle(spa_plan *plan, void *ws, uint8_t handle[SPA_IPC_HANDLE_BYTES]) {
    if (!plan || !ws || !handle) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->comm->kind != KIND_P2P) return fail(SPA_ERR_INVALID, "not a p2p plan");
    SPA_CHECK_CUDA(cudaSetDevice(plan->comm->device));
    CUdeviceptr base = 0;
    size_t size = 0;
    if (drv().range(&base, &size, reinterpret_cast<CUdeviceptr>(ws)) != CUDA_SUCCESS)
        return fail(SPA_ERR_INVALID, "ws is not device memory");
    size_t need = 0;
    SPA_TRY(spa_plan_workspace_bytes(plan, &need));
    const unsigned long long off = reinterpret_cast<CUdeviceptr>(ws) - base;
    if (off + need > size) return fail(SPA_ERR_INVALID, "ws allocation smaller than the plan's workspace");
    cudaIpcMemHandle_t h;
    SPA_CHECK_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
    static_assert(sizeof(h) + 8 == SPA_IPC_HANDLE_BYTES, "handle size");
    memcpy(handle, &h, sizeof(h));
    memcpy(handle + sizeof(h), &off, 8);
    return SPA_OK;
}

spa_status spa_plan_ipc_open(spa_plan *plan, void *ws, const uint8_t *handles) {
    if (!plan || !ws || !handles) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->comm->kind != KIND_P2P) return fail(SPA_ERR_INVALID, "not a p2p plan");
    if (!plan->peer_ws.empty()) return fail(SPA_ERR_INVALID, "p2p plan already opened");
    SPA_CHECK_CUDA(cudaSetDevice(plan->comm->device));
    const int me = plan->comm->rank;
    std::vector<uint8_t *> peers(plan->P, nullptr);
    for (int q = 0; q < plan->P; ++q) {
        if (q == me) {
            peers[q] = reinterpret_cast<uint8_t *>(ws);
            continue;
        }
        cudaIpcMemHandle_t h;
        unsigned long long off = 0;
        memcpy(&h, handles + (size_t)q * SPA_IPC_HANDLE_BYTES, sizeof(h));
        memcpy(&off, handles + (size_t)q * SPA_IPC_HANDLE_BYTES + sizeof(h), 8);
        void *base = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (void *b : plan->ipc_bases) cudaIpcCloseMemHandle(b);
            plan->ipc_bases.clear();
            return fail(SPA_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
        }
        peers[q] = reinterpret_cast<uint8_t *>(base) + off;
        plan->ipc_bases.push_back(base);
    }
    int flush = 0;
    if (cudaDeviceGetAttribute(&flush, static_cast<cudaDeviceAttr>(CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES),
                               plan->comm->device) == cudaSuccess)
        plan->p2p_flush = flush != 0;
    cudaGetLastError();
    plan->peer_ws = peers;
    plan->epoch = 0;
    if (plan->U > 1) {   // USP: the sub-plans' peers are the group's / ring's ranks, at the sub-plan offsets
        const int U = plan->U, R = plan->R, u = me % U, rho = me / U;
        spa_plan *up = plan->uly_plan, *rp = plan->ring_plan;
        up->peer_ws.assign(U, nullptr);
        rp->peer_ws.assign(R, nullptr);
        for (int i = 0; i < U; ++i) up->peer_ws[i] = peers[rho * U + i] + plan->off_parts;
        for (int i = 0; i < R; ++i) rp->peer_ws[i] = peers[i * U + u] + plan->off_ring_ws;
        up->epoch = rp->epoch = 0;
        up->p2p_flush = rp->p2p_flush = plan->p2p_flush;
        if (up->P > 1)
            SPA_CHECK_CUDA(cudaMemset(up->peer_ws[u] + up->off_flags, 0, (size_t)flag_bytes(up)));
        if (rp->P > 1)
            SPA_CHECK_CUDA(cudaMemset(rp->peer_ws[rho] + rp->off_flags, 0, (size_t)flag_bytes(rp)));
        return SPA_OK;
    }
    // this rank's flags start at 0 (the caller synchronises all ranks after ipc_open, before the first call)
    SPA_CHECK_CUDA(cudaMemset(reinterpret_cast<uint8_t *>(ws) + plan->off_flags, 0, (size_t)flag_bytes(plan)));
    return SPA_OK;
}

// ------------------------------------------------------------------ NCCL symmetric windows (SURVEY f1 on NCCL plans)
spa_status spa_mem_alloc(size_t bytes, void **ptr) {
    if (!ptr || bytes == 0) return fail(SPA_ERR_INVALID, "spa_mem_alloc: NULL ptr or 0 bytes");
    *ptr = nullptr;
    SPA_CHECK_NCCL(ncclMemAlloc(ptr, bytes));
    return SPA_OK;
}

spa_status spa_mem_free(void *ptr) {
    if (!ptr) return SPA_OK;
    SPA_CHECK_NCCL(ncclMemFree(ptr));
    return SPA_OK;
}

spa_status spa_plan_window_register(spa_plan *plan, void *ws) {
    if (!plan || !ws) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->comm->kind != KIND_NCCL || !plan->comm->nccl) return fail(SPA_ERR_INVALID, "not an NCCL plan");
    if (plan->ring || plan->U > 1)
        return fail(SPA_ERR_UNSUPPORTED, "NCCL window: Ulysses / PipeSP / Aco plans (ring plans exchange with NCCL)");
    if (plan->win) return fail(SPA_ERR_INVALID, "NCCL window already registered");
    if (plan->P == 1) return SPA_OK;   // nothing is exchanged
    if (reinterpret_cast<uintptr_t>(ws) % NCCL_WIN_REQUIRED_ALIGNMENT)
        return fail(SPA_ERR_INVALID, "NCCL window: ws must be 4096-byte aligned (spa_mem_alloc)");
    SPA_CHECK_CUDA(cudaSetDevice(plan->comm->device));
    // every rank must be in this rank's NVLink domain, with LSA index = world rank (the peer addresses below)
    int lsa_size = 0, lsa_rank = -1;
    SPA_CHECK_NCCL(nccl_lsa_team(plan->comm->nccl, &lsa_size, &lsa_rank));
    if (lsa_size != plan->comm->nranks || lsa_rank != plan->comm->rank)
        return fail(SPA_ERR_UNSUPPORTED, "NCCL window: the ranks do not form one NVLink domain (LSA team " +
                                             std::to_string(lsa_size) + " of " + std::to_string(plan->comm->nranks) + ")");
    const size_t bytes = (size_t)align_up(plan->ws_rank_bytes, NCCL_WIN_REQUIRED_ALIGNMENT);
    ncclWindow_t w = nullptr;
    SPA_CHECK_NCCL(ncclCommWindowRegister(plan->comm->nccl, ws, bytes, &w, NCCL_WIN_COLL_SYMMETRIC));
    std::vector<uint8_t *> peers(plan->P, nullptr);
    cudaStream_t st = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = nccl_window_bases(w, plan->P, peers.data(), st);
    if (st) cudaStreamDestroy(st);
    if (e != cudaSuccess) {
        ncclCommWindowDeregister(plan->comm->nccl, w);
        return fail(SPA_ERR_CUDA, std::string("NCCL window: resolving the peers' addresses: ") + cudaGetErrorString(e));
    }
    for (uint8_t *b : peers)
        if (!b) {
            ncclCommWindowDeregister(plan->comm->nccl, w);
            return fail(SPA_ERR_COMM, "NCCL window: a rank is outside this NVLink domain (no LSA address)");
        }
    plan->win = w;
    plan->peer_ws = peers;
    plan->peer_ws[plan->comm->rank] = reinterpret_cast<uint8_t *>(ws);   // local calls use the caller's address
    plan->epoch = 0;
    int flush = 0;
    if (cudaDeviceGetAttribute(&flush, static_cast<cudaDeviceAttr>(CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES),
                               plan->comm->device) == cudaSuccess)
        plan->p2p_flush = flush != 0;
    cudaGetLastError();
    // this rank's flags start at 0 (the caller synchronises all ranks after the registration, before the first call)
    SPA_CHECK_CUDA(cudaMemset(reinterpret_cast<uint8_t *>(ws) + plan->off_flags, 0, (size_t)flag_bytes(plan)));
    return SPA_OK;
}

spa_status spa_comm_window_selftest(spa_comm *comm, size_t bytes) {
    if (!comm || comm->kind != KIND_NCCL || !comm->nccl) return fail(SPA_ERR_INVALID, "not an NCCL comm");
    if (bytes < 4096 || bytes % 4096) return fail(SPA_ERR_INVALID, "bytes: a positive multiple of 4096");
    SPA_CHECK_CUDA(cudaSetDevice(comm->device));
    int lsa_size = 0, lsa_rank = -1;
    SPA_CHECK_NCCL(nccl_lsa_team(comm->nccl, &lsa_size, &lsa_rank));
    if (lsa_size != comm->nranks || lsa_rank != comm->rank)
        return fail(SPA_ERR_UNSUPPORTED, "window self-test: the LSA team is not the whole communicator");
    void *buf = nullptr;
    SPA_CHECK_NCCL(ncclMemAlloc(&buf, bytes));
    ncclWindow_t w = nullptr;
    spa_status rc = SPA_OK;
    ncclResult_t r = ncclCommWindowRegister(comm->nccl, buf, bytes, &w, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
        ncclMemFree(buf);
        return fail(SPA_ERR_COMM, std::string("ncclCommWindowRegister: ") + ncclGetErrorString(r));
    }
    std::vector<uint8_t *> bases(comm->nranks, nullptr);
    cudaStream_t st = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = nccl_window_bases(w, comm->nranks, bases.data(), st);
    std::vector<uint32_t> host(bytes / 4);
    if (e == cudaSuccess) e = nccl_window_fill_pattern(reinterpret_cast<uint32_t *>(bases[comm->rank]),
                                                       (long long)(bytes / 4), 0x5eedu + comm->rank, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(host.data(), buf, bytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (st) cudaStreamDestroy(st);
    if (e != cudaSuccess) {
        rc = fail(SPA_ERR_CUDA, std::string("window self-test: ") + cudaGetErrorString(e));
    } else {
        for (size_t i = 0; i < host.size(); ++i)
            if (host[i] != (((uint32_t)(i * 2654435761u)) ^ (0x5eedu + (uint32_t)comm->rank))) {
                rc = fail(SPA_ERR_COMM, "window self-test: a store through the rank's LSA address is not visible locally");
                break;
            }
    }
    ncclCommWindowDeregister(comm->nccl, w);
    ncclMemFree(buf);
    return rc;
}

spa_status spa_comm_init_host(spa_comm **comm, int nranks, int rank) {
    if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(SPA_ERR_INVALID, "bad host comm arguments");
    spa_comm *c = new spa_comm;
    c->kind = KIND_HOST; c->nranks = nranks; c->rank = rank;
    *comm = c;
    return SPA_OK;
}

spa_status spa_comm_split(spa_comm *comm, int color, int key, spa_comm **sub) {
    if (!comm || !sub) return fail(SPA_ERR_INVALID, "NULL argument");
    if (comm->kind != KIND_NCCL) return fail(SPA_ERR_UNSUPPORTED, "split needs an NCCL comm");
    ncclComm_t nc = nullptr;
    SPA_CHECK_NCCL(ncclCommSplit(comm->nccl, color < 0 ? NCCL_SPLIT_NOCOLOR : color, key, &nc, nullptr));
    if (color < 0 || !nc) {
        *sub = nullptr;
        return SPA_OK;
    }
    spa_comm *c = new spa_comm;
    c->kind = KIND_NCCL; c->device = comm->device; c->nccl = nc;
    SPA_CHECK_NCCL(ncclCommCount(nc, &c->nranks));
    SPA_CHECK_NCCL(ncclCommUserRank(nc, &c->rank));
    *sub = c;
    return SPA_OK;
}

spa_status spa_comm_check(spa_comm *comm) {
    if (!comm) return fail(SPA_ERR_INVALID, "comm is NULL");
    if (comm->kind == KIND_NCCL) {
        ncclResult_t a = ncclSuccess;
        SPA_CHECK_NCCL(ncclCommGetAsyncError(comm->nccl, &a));
        if (a != ncclSuccess && a != ncclInProgress) return fail(SPA_ERR_COMM, ncclGetErrorString(a));
    }
    if (comm->kind != KIND_HOST) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(SPA_ERR_CUDA, cudaGetErrorString(e));
    }
    return SPA_OK;
}

spa_status spa_comm_wait(spa_comm *comm, void *stream, int timeout_ms) {
    if (!comm) return fail(SPA_ERR_INVALID, "comm is NULL");
    if (comm->kind == KIND_HOST) return fail(SPA_ERR_UNSUPPORTED, "host-only comm");
    SPA_CHECK_CUDA(cudaSetDevice(comm->device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) return fail(SPA_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(q));
        if (comm->kind == KIND_NCCL) {
            ncclResult_t a = ncclSuccess;
            SPA_CHECK_NCCL(ncclCommGetAsyncError(comm->nccl, &a));
            if (a != ncclSuccess && a != ncclInProgress) {
                ncclCommAbort(comm->nccl);   // a peer failed: unblock this rank's kernels
                comm->nccl = nullptr;
                return fail(SPA_ERR_COMM, std::string("communicator failed, aborted: ") + ncclGetErrorString(a));
            }
        }
        const long long ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
        if (timeout_ms >= 0 && ms > timeout_ms) {
            if (comm->kind == KIND_NCCL && comm->nccl) {
                ncclCommAbort(comm->nccl);
                comm->nccl = nullptr;
                return fail(SPA_ERR_COMM, "timeout: communicator aborted (a peer stopped participating)");
            }
            return fail(SPA_ERR_COMM, "timeout waiting for the stream");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    return SPA_OK;
}

spa_status spa_comm_destroy(spa_comm *comm) {
    if (!comm) return SPA_OK;
    if (comm->stream) cudaStreamDestroy(comm->stream);
    if (comm->nccl) ncclCommDestroy(comm->nccl);
    delete comm;
    return SPA_OK;
}

spa_status spa_comm_info(const spa_comm *comm, int *nranks, int *rank, int *kind) {
    if (!comm) return fail(SPA_ERR_INVALID, "comm is NULL");
    if (nranks) *nranks = comm->nranks;
    if (rank) *rank = comm->rank;
    if (kind) *kind = comm->kind;
    return SPA_OK;
}

spa_status spa_plan_create(spa_plan **plan, spa_comm *comm, const spa_shape *shape) {
    if (!plan || !comm || !shape) return fail(SPA_ERR_INVALID, "NULL argument");
    const spa_shape &s = *shape;
    if (s.B < 1 || s.S < 1 || s.H < 1) return fail(SPA_ERR_SHAPE, "B, S, H must be >= 1");
    if (s.D != 64 && s.D != 96 && s.D != 128) return fail(SPA_ERR_UNSUPPORTED, "D must be 64, 96 or 128");
    if (s.stages < 1) return fail(SPA_ERR_SHAPE, "stages must be >= 1");
    const int P = comm->nranks;
    const int Psrc = s.n_src == 0 ? P : s.n_src;
    if (Psrc < 1 || Psrc > P) return fail(SPA_ERR_SHAPE, "n_src must be in [0, nranks]");
    if (s.S < Psrc) return fail(SPA_ERR_SHAPE, "fewer tokens than source ranks");
    if (s.pad_heads != 0 && s.pad_heads != 1) return fail(SPA_ERR_INVALID, "pad_heads must be 0 or 1");
    if (s.ring != 0 && s.ring != 1) return fail(SPA_ERR_INVALID, "ring must be 0 or 1");
    if (s.ulysses < 0 || (!s.ring && s.ulysses > 1)) return fail(SPA_ERR_INVALID, "ulysses degree needs ring = 1");
    if (s.ring && (s.stages != 1 || s.pad_heads != 0))
        return fail(SPA_ERR_INVALID, "ring / USP plans take stages = 1 and pad_heads = 0");
    if (s.ring && s.ulysses > 1) return create_usp_plan(plan, comm, s);
    if (s.ring) {
        // Ring attention: every rank keeps all heads; only S % P matters.
        if (s.n_src != 0 && s.n_src != P) return fail(SPA_ERR_SHAPE, "ring plans have no co-processor ranks");
        if (s.S % P) return fail(SPA_ERR_SHAPE, "S must be divisible by nranks");
        spa_plan *p = new spa_plan;
        p->comm = comm; p->sh = s; p->P = P; p->Psrc = P; p->ring = true;
        p->Hp = s.H; p->h = s.H; p->S_l = s.S / P;
        p->split = make_split(1, p->S_l, 1);
        p->E_loc = (long long)s.B * p->S_l * s.H * s.D;
        long long off = 0;
        auto take = [&](long long bytes) { long long o = off; off = align_up(off + bytes, 256); return o; };
        if (P > 1) {
            p->off_kvbuf = take(4 * p->E_loc * 2);                        // [slot 0/1][K/V] bf16
            p->off_parts = take((long long)P * p->E_loc * 4);             // [P] fp32 partial O
            p->off_lse = take((long long)P * (p->E_loc / s.D) * 4);       // [P] fp32 lse
            if (comm->kind == KIND_P2P) {   // ring steps' arrival / slot-free flags
                p->n_flag_stages = P;
                p->off_flags = take(flag_bytes(p));
            }
        }
        p->ws_rank_bytes = off;
        *plan = p;
        return SPA_OK;
    }
    if (s.H % P && !s.pad_heads)
        return fail(SPA_ERR_SHAPE, "H must be divisible by nranks (or set shape.pad_heads = 1)");
    spa_plan *p = new spa_plan;
    p->comm = comm; p->sh = s; p->P = P; p->Psrc = Psrc;
    p->Hp = (s.H + P - 1) / P * P;
    p->h = p->Hp / P;
    // sequence shards differ by at most one token: the first S % Psrc source ranks hold one more (R9)
    p->len.resize(Psrc);
    p->start.resize(Psrc + 1);
    p->start[0] = 0;
    for (int r = 0; r < Psrc; ++r) {
        p->len[r] = s.S / Psrc + (r < s.S % Psrc ? 1 : 0);
        p->start[r + 1] = p->start[r] + p->len[r];
    }
    p->S_l = p->len[0];   // the longest shard (buffer sizing)
    p->split = make_split(p->h, p->S_l, s.stages);
    if (p->split.C > p->len[Psrc - 1]) {
        delete p;
        return fail(SPA_ERR_SHAPE, "more query chunks than local tokens");
    }
    p->E_src = (long long)s.B * p->S_l * p->Hp * s.D;   // send / orecv: all (padded) head groups
    p->E_own = (long long)s.B * s.S * p->h * s.D;
    if (P > 1) {
        long long off = 0;
        auto take = [&](long long elems) { long long o = off; off = align_up(off + elems * 2, 256); return o; };
        p->off_sendQ = take(p->E_src); p->off_sendK = take(p->E_src); p->off_sendV = take(p->E_src);
        p->off_orecv = take(p->E_src);
        p->off_recvQ = take(p->E_own); p->off_recvK = take(p->E_own); p->off_recvV = take(p->E_own);
        p->off_O = take(p->E_own);
        if (comm->kind != KIND_LOOPBACK) {   // epoch flags + the direct transport's output landing buffer (P2P plans;
                                             // NCCL plans once a symmetric window is registered)
            p->n_flag_stages = p->split.n();
            p->off_flags = take((flag_bytes(p) + 1) / 2);
            p->off_outbuf = take((long long)s.B * p->S_l * s.H * s.D);
        }
        p->ws_rank_bytes = off;
    }
    *plan = p;
    return SPA_OK;
}

spa_status spa_plan_workspace_bytes(const spa_plan *plan, size_t *bytes) {
    if (!plan || !bytes) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->ws_total >= 0) {
        *bytes = (size_t)plan->ws_total;
        return SPA_OK;
    }
    long long per = plan->ws_rank_bytes;
    *bytes = (size_t)(plan->comm->kind == KIND_LOOPBACK ? per * plan->P : per);
    return SPA_OK;
}

spa_status spa_plan_stage_split(const spa_plan *plan, int *G_h, int *C, int *g) {
    if (!plan) return fail(SPA_ERR_INVALID, "plan is NULL");
    if (G_h) *G_h = plan->split.G_h;
    if (C) *C = plan->split.C;
    if (g) *g = plan->split.g;
    return SPA_OK;
}

spa_status spa_plan_destroy(spa_plan *plan) {
    if (!plan) return SPA_OK;
    spa_plan_destroy(plan->uly_plan);
    spa_plan_destroy(plan->ring_plan);
    if (plan->uly_comm) spa_comm_destroy(plan->uly_comm);
    if (plan->ring_comm) spa_comm_destroy(plan->ring_comm);
    for (void *b : plan->ipc_bases) cudaIpcCloseMemHandle(b);
    if (plan->win && plan->comm->nccl) ncclCommWindowDeregister(plan->comm->nccl, plan->win);
    for (auto e : plan->sync_ev) cudaEventDestroy(e);
    for (auto e : plan->prof_ev) cudaEventDestroy(e);
    if (plan->sc_alt) cudaStreamDestroy(plan->sc_alt);
    for (cudaStream_t st : plan->extra_streams) cudaStreamDestroy(st);
    if (plan->s_h2d) cudaStreamDestroy(plan->s_h2d);
    if (plan->s_d2h) cudaStreamDestroy(plan->s_d2h);
    delete plan;
    return SPA_OK;
}

spa_status spa_plan_set_option(spa_plan *plan, int option, int value) {
    if (!plan) return fail(SPA_ERR_INVALID, "plan is NULL");
    if (plan->U > 1 && (option == SPA_OPT_PROFILE || option == SPA_OPT_SKIP_COMM)) {   // USP: the sub-plans too
        SPA_TRY(spa_plan_set_option(plan->uly_plan, option, value));
        SPA_TRY(spa_plan_set_option(plan->ring_plan, option, value));
    }
    switch (option) {
        case SPA_OPT_PROFILE: plan->profile = value != 0; break;
        case SPA_OPT_SKIP_COMM: plan->skip_comm = value != 0; break;
        case SPA_OPT_COPROC_BUSY: plan->coproc_busy = value != 0; break;
        case SPA_OPT_RANK_ONLY:
            if (plan->comm->kind != KIND_LOOPBACK || value < 0 || value > plan->P)
                return fail(SPA_ERR_INVALID, "rank-only mode: loopback plans, value = rank + 1 (0 = off)");
            plan->rank_only = value - 1;
            break;
        case SPA_OPT_LOOPBACK_CE:
            if (plan->comm->kind != KIND_LOOPBACK) return fail(SPA_ERR_INVALID, "loopback plans only");
            plan->loopback_ce = value != 0;
            break;
        case SPA_OPT_STAGE_WINDOW:
            if (value < 1 || value > 8) return fail(SPA_ERR_INVALID, "stage window must be in [1, 8]");
            plan->stage_window = value;
            break;
        case SPA_OPT_COMM_SMS:
            if (value < 0 || value > 64) return fail(SPA_ERR_INVALID, "comm SMs must be in [0, 64]");
            plan->comm_sms = value;
            break;
        case SPA_OPT_DIRECT:
            if (value && (plan->ring || plan->Psrc > kMaxDst))
                return fail(SPA_ERR_UNSUPPORTED, "direct transport: PipeSP / Ulysses / Aco plans with <= 16 sources");
            plan->direct = value != 0;
            break;
        default: return fail(SPA_ERR_INVALID, "unknown option");
    }
    return SPA_OK;
}

spa_status spa_plan_set_kv_len(spa_plan *plan, const int32_t *kv_len) {
    if (!plan) return fail(SPA_ERR_INVALID, "plan is NULL");
    if (kv_len && reinterpret_cast<uintptr_t>(kv_len) % 4) return fail(SPA_ERR_INVALID, "kv_len not 4-byte aligned");
    plan->kv_len = kv_len;
    return SPA_OK;
}

spa_status spa_plan_last_profile(spa_plan *plan, spa_profile *out) {
    if (!plan || !out) return fail(SPA_ERR_INVALID, "NULL argument");
    if (!plan->have_profile) return fail(SPA_ERR_INVALID, "no profiled call yet (set SPA_OPT_PROFILE)");
    spa_profile r{};
    auto span = [&](const std::string &nm, float *dst) -> spa_status {
        auto b = plan->prof_idx.find(nm + "#b"), e = plan->prof_idx.find(nm + "#e");
        if (b == plan->prof_idx.end() || e == plan->prof_idx.end()) return SPA_OK;
        cudaError_t err = cudaEventElapsedTime(dst, plan->prof_ev[b->second], plan->prof_ev[e->second]);
        if (err != cudaSuccess) return fail(SPA_ERR_CUDA, std::string("profile: ") + cudaGetErrorString(err));
        return SPA_OK;
    };
    const int N = plan->prof_stages;
    r.n_stages = N;
    SPA_TRY(span("total", &r.total_ms));
    SPA_TRY(span("pack", &r.pack_ms));
    SPA_TRY(span("unpack", &r.unpack_ms));
    for (int k = 0; k < N && k < 64; ++k) {
        SPA_TRY(span("attn" + std::to_string(k), &r.attn_ms[k]));
        SPA_TRY(span("in" + std::to_string(k), &r.a2a_in_ms[k]));
        SPA_TRY(span("out" + std::to_string(k), &r.a2a_out_ms[k]));
    }
    r.attn_launches = plan->attn_launches;
    r.copy_launches = plan->copy_launches;
    r.gemm_launches = plan->gemm_launches;
    if (plan->U > 1 && plan->ring_plan->have_profile) {   // USP: the ring sub-plan's (last) call is the attention
        spa_profile rp{};
        SPA_TRY(spa_plan_last_profile(plan->ring_plan, &rp));
        r.attn_ms[0] = rp.total_ms;
        r.attn_launches = rp.attn_launches;
        r.copy_launches = rp.copy_launches;
    }
    *out = r;
    return SPA_OK;
}

spa_status spa_ulysses_attention(spa_plan *plan, const void *q, const void *k, const void *v, void *out, void *ws,
                                 void *stream) {
    if (plan && plan->Psrc != plan->P) return fail(SPA_ERR_INVALID, "Aco plan: use spa_aco_attention");
    return attention_call(plan, 1, &q, &k, &v, &out, ws, stream, false, true);
}
spa_status spa_pipesp_attention(spa_plan *plan, const void *q, const void *k, const void *v, void *out, void *ws,
                                void *stream) {
    if (plan && plan->Psrc != plan->P) return fail(SPA_ERR_INVALID, "Aco plan: use spa_aco_attention");
    return attention_call(plan, 1, &q, &k, &v, &out, ws, stream, false, false);
}
spa_status spa_aco_attention(spa_plan *plan, const void *q, const void *k, const void *v, void *out, void *ws,
                             void *stream) {
    if (!plan) return fail(SPA_ERR_INVALID, "plan is NULL");
    if (plan->ring) return fail(SPA_ERR_INVALID, "ring plan: use spa_ring_attention");
    // no co-processor ranks (N_decode = 0): Aco is PipeSP on all ranks
    if (plan->Psrc == plan->P) return attention_call(plan, 1, &q, &k, &v, &out, ws, stream, false, false);
    if (plan->coproc_busy) return fail(SPA_ERR_BUSY, "co-processor group busy");
    const bool src = plan->comm->kind != KIND_LOOPBACK && is_source(plan, plan->comm->rank);
    if (!src) {
        if (q || k || v || out) return fail(SPA_ERR_INVALID, "co-processor ranks pass NULL q/k/v/out");
        Exec x{};
        SPA_TRY(prepare(plan, x, ws, stream, false));
        x.s = &plan->split;
        return execute(x);
    }
    return attention_call(plan, 1, &q, &k, &v, &out, ws, stream, false, false);
}

spa_status spa_ulysses_attention_local(spa_plan *plan, const void *const q[], const void *const k[],
                                       const void *const v[], void *const out[], void *ws, void *stream) {
    if (!plan || !q || !k || !v || !out) return fail(SPA_ERR_INVALID, "NULL argument");
    return attention_call(plan, n_local_srcs(plan), q, k, v, out, ws, stream, true, true);
}
spa_status spa_pipesp_attention_local(spa_plan *plan, const void *const q[], const void *const k[],
                                      const void *const v[], void *const out[], void *ws, void *stream) {
    if (!plan || !q || !k || !v || !out) return fail(SPA_ERR_INVALID, "NULL argument");
    return attention_call(plan, n_local_srcs(plan), q, k, v, out, ws, stream, true, false);
}
spa_status spa_aco_attention_local(spa_plan *plan, const void *const q[], const void *const k[],
                                   const void *const v[], void *const out[], void *ws, void *stream) {
    if (!plan || !q || !k || !v || !out) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->Psrc != plan->P && plan->coproc_busy) return fail(SPA_ERR_BUSY, "co-processor group busy");
    return attention_call(plan, n_local_srcs(plan), q, k, v, out, ws, stream, true, false);
}

// ------------------------------------------------------------------ QKV projection fused with PipeSP
static spa_status qkv_check(const spa_plan *p, int C) {
    if (!p) return fail(SPA_ERR_INVALID, "plan is NULL");
    if (p->ring) return fail(SPA_ERR_UNSUPPORTED, "QKV projection calls need a Ulysses / PipeSP plan");
    if (p->Psrc != p->P || p->Hp != p->sh.H)
        return fail(SPA_ERR_UNSUPPORTED, "QKV projection calls: no co-processor ranks, no head padding");
    if (C < 8 || C % 8) return fail(SPA_ERR_SHAPE, "hidden dim C must be a positive multiple of 8");
    return SPA_OK;
}

spa_status spa_plan_qkv_weight_bytes(const spa_plan *plan, int C, size_t *bytes) {
    SPA_TRY(qkv_check(plan, C));
    if (!bytes) return fail(SPA_ERR_INVALID, "NULL argument");
    *bytes = (size_t)qkv_packed_bytes(plan, C);
    return SPA_OK;
}

spa_status spa_plan_qkv_workspace_bytes(const spa_plan *plan, size_t *bytes) {
    if (!plan || !bytes) return fail(SPA_ERR_INVALID, "NULL argument");
    SPA_TRY(qkv_check(plan, 8));
    if (plan->P == 1) *bytes = (size_t)3 * plan->sh.B * plan->sh.S * plan->sh.H * plan->sh.D * 2;
    else return spa_plan_workspace_bytes(plan, bytes);
    return SPA_OK;
}

spa_status spa_plan_pack_qkv_weight(spa_plan *plan, int C, const void *w, const float *bias, void *w_packed,
                                    void *stream) {
    SPA_TRY(qkv_check(plan, C));
    SPA_TRY(check_ptr(w, "w"));
    SPA_TRY(check_ptr(w_packed, "w_packed"));
    if (bias && reinterpret_cast<uintptr_t>(bias) % 16) return fail(SPA_ERR_INVALID, "bias not 16-byte aligned");
    if (plan->comm->kind != KIND_HOST) SPA_CHECK_CUDA(cudaSetDevice(plan->comm->device));
    else return fail(SPA_ERR_UNSUPPORTED, "host-only comm cannot execute");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const Split &s = plan->split;
    const long long gD = (long long)s.g * plan->sh.D, H = plan->sh.H, D = plan->sh.D, h = plan->h, P = plan->P;
    uint8_t *wp = reinterpret_cast<uint8_t *>(w_packed);
    // weight rows: [kh][t][q] runs of g*D rows of W (row t*H*D + (q*h + kh*g)*D)
    std::vector<CopyJob> jobs(1);
    CopyJob &j = jobs[0];
    j.src = reinterpret_cast<const uint8_t *>(w);
    j.dst = wp;
    j.count[0] = s.G_h; j.count[1] = 3; j.count[2] = P; j.count[3] = 1;
    j.src_stride[0] = gD * C * 2; j.src_stride[1] = H * D * C * 2; j.src_stride[2] = h * D * C * 2;
    j.dst_stride[0] = 3 * P * gD * C * 2; j.dst_stride[1] = P * gD * C * 2; j.dst_stride[2] = gD * C * 2;
    j.run_bytes = gD * C * 2;
    int launches = 0;
    if (bias) {   // the same column permutation on the fp32 bias
        CopyJob b = j;
        b.src = reinterpret_cast<const uint8_t *>(bias);
        b.dst = wp + qkv_bias_off(plan, C);
        b.src_stride[0] = gD * 4; b.src_stride[1] = H * D * 4; b.src_stride[2] = h * D * 4;
        b.dst_stride[0] = 3 * P * gD * 4; b.dst_stride[1] = P * gD * 4; b.dst_stride[2] = gD * 4;
        b.run_bytes = gD * 4;
        jobs.push_back(b);
    } else {
        SPA_CHECK_CUDA(cudaMemsetAsync(wp + qkv_bias_off(plan, C), 0, (size_t)s.G_h * qkv_cols(plan) * 4, st));
    }
    SPA_CHECK_CUDA(launch_copy_jobs(jobs.data(), (int)jobs.size(), st, &launches));
    return SPA_OK;
}

static spa_status qkv_call(spa_plan *p, int C, int n, const void *const x[], const void *w_packed, void *const out[],
                           void *ws, void *stream, bool local) {
    SPA_TRY(qkv_check(p, C));
    SPA_TRY(check_ptr(w_packed, "w_packed"));
    Exec e{};
    SPA_TRY(prepare(p, e, ws, stream, local));
    if (p->P == 1) SPA_TRY(check_ptr(ws, "ws"));
    e.s = &p->split;
    e.qkv = true;
    e.wp = reinterpret_cast<const uint8_t *>(w_packed);
    e.C = C;
    for (int i = 0; i < n; ++i) {
        SPA_TRY(check_ptr(x[i], "x"));
        SPA_TRY(check_ptr(out[i], "out"));
        e.xin.push_back(x[i]);
        e.ptr.q.push_back(nullptr); e.ptr.k.push_back(nullptr); e.ptr.v.push_back(nullptr);
        e.ptr.out.push_back(out[i]);
    }
    return execute(e);
}

spa_status spa_pipesp_qkv_attention(spa_plan *plan, int C, const void *x, const void *w_packed, void *out, void *ws,
                                    void *stream) {
    return qkv_call(plan, C, 1, &x, w_packed, &out, ws, stream, false);
}

spa_status spa_pipesp_qkv_attention_local(spa_plan *plan, int C, const void *const x[], const void *w_packed,
                                          void *const out[], void *ws, void *stream) {
    if (!plan || !x || !out) return fail(SPA_ERR_INVALID, "NULL argument");
    return qkv_call(plan, C, n_local_srcs(plan), x, w_packed, out, ws, stream, true);
}

spa_status spa_qkv_projection(spa_plan *plan, int C, int rank, const void *x, const void *w_packed, void *q, void *k,
                              void *v, void *stream) {
    SPA_TRY(qkv_check(plan, C));
    if (plan->comm->kind == KIND_HOST) return fail(SPA_ERR_UNSUPPORTED, "host-only comm cannot execute");
    if (rank < 0 || rank >= plan->P || (plan->comm->kind == KIND_NCCL && rank != plan->comm->rank))
        return fail(SPA_ERR_INVALID, "bad rank");
    for (const void *ptr : {x, w_packed, (const void *)q, (const void *)k, (const void *)v}) SPA_TRY(check_ptr(ptr, "pointer"));
    SPA_CHECK_CUDA(cudaSetDevice(plan->comm->device));
    const Split &s = plan->split;
    plan->gemm_launches = 0;
    for (int kh = 0; kh < s.G_h; ++kh) {   // head group kh: heads q*h + kh*g + jj of the [B, S_r, H, D] outputs
        const long long off = (long long)kh * s.g * plan->sh.D * 2;
        void *dst[3] = {(uint8_t *)q + off, (uint8_t *)k + off, (uint8_t *)v + off};
        SPA_TRY(launch_qkv(plan, x, reinterpret_cast<const uint8_t *>(w_packed), C, rank, kh, dst,
                           (long long)plan->h * plan->sh.D, (long long)plan->sh.H * plan->sh.D,
                           reinterpret_cast<cudaStream_t>(stream)));
    }
    return SPA_OK;
}

// ------------------------------------------------------------------ ring attention (R21)
// Rank r keeps its query shard and all heads; at step t it attends to the K/V shard of rank (r - t) mod P, which
// travels the ring r-1 -> r -> r+1 on the comm stream while the previous block is being computed (double-buffered
// receive slots); every step writes an fp32 partial O and its per-row lse, and lse_merge combines the P partials.
static AttnProblem ring_problem(const spa_plan *p, const void *q, const void *k, const void *v, float *o32,
                                float *lse, int kv_src = 0) {
    AttnProblem a{};
    const long long tok = (long long)p->sh.H * p->sh.D;
    a.q = q; a.k = k; a.v = v; a.o = nullptr; a.o32 = o32; a.lse = lse;
    a.B = p->sh.B; a.Sq = a.Skv = p->S_l; a.n_heads = p->sh.H; a.D = p->sh.D;
    a.q_tok_stride = a.kv_tok_stride = a.o_tok_stride = tok;
    a.q_batch_stride = a.kv_batch_stride = a.o_batch_stride = (long long)p->S_l * tok;
    a.kv_len = p->kv_len;   // key-padding mask by global position: this block's keys start at kv_src * S_l
    a.kv_offset = kv_src * p->S_l;
    return a;
}

static spa_status ring_call(spa_plan *p, int n, const void *const q[], const void *const k[], const void *const v[],
                            void *const out[], void *ws, void *stream, bool local) {
    if (!p) return fail(SPA_ERR_INVALID, "plan is NULL");
    NvtxRange range("spa: ring attention");
    if (!p->ring) return fail(SPA_ERR_INVALID, "not a ring plan (shape.ring = 1)");
    if (p->U > 1) {
        // the ring runs over the Ulysses groups, whose token blocks are contiguous in the global sequence
        SPA_TRY(spa_plan_set_kv_len(p->ring_plan, p->kv_len));
        return usp_call(p, q, k, v, out, ws, stream, local);
    }
    Exec x{};
    SPA_TRY(prepare(p, x, ws, stream, local));
    for (int i = 0; i < n; ++i) {
        SPA_TRY(check_ptr(q[i], "q")); SPA_TRY(check_ptr(k[i], "k"));
        SPA_TRY(check_ptr(v[i], "v")); SPA_TRY(check_ptr(out[i], "out"));
    }
    p->attn_launches = 0;
    p->copy_launches = 0;
    const int P = p->P;
    const long long tok = (long long)p->sh.H * p->sh.D;
    cudaStream_t sc = x.sc;
    SPA_TRY(ensure_events(p, 4 + 2 * (size_t)P, p->profile ? 8 + 4 * (size_t)P : 0));
    Prof pr{p};
    pr.begin("total", sc);
    if (P == 1) {   // one block: the plain kernel
        AttnProblem a = ring_problem(p, q[0], k[0], v[0], nullptr, nullptr);
        a.o = out[0]; a.o32 = nullptr;
        pr.begin("attn0", sc);
        SPA_CHECK_CUDA(launch_attention(a, sc));
        pr.end("attn0", sc);
        ++p->attn_launches;
        pr.end("total", sc);
        finish_profile(p, pr, 1);
        return SPA_OK;
    }
    const long long rows = p->E_loc / p->sh.D;
    auto parts = [&](int r) { return reinterpret_cast<float *>(resolve(x, r, BUF_WS, p->off_parts)); };
    auto lses = [&](int r) { return reinterpret_cast<float *>(resolve(x, r, BUF_WS, p->off_lse)); };
    auto merge = [&](int r, void *o) -> spa_status {
        SPA_CHECK_CUDA(launch_lse_merge(parts(r), p->E_loc, lses(r), rows, P, p->sh.B, p->S_l, p->sh.H, p->sh.D, o,
                                        tok, (long long)p->S_l * tok, sc));
        ++p->copy_launches;
        return SPA_OK;
    };
    if (p->comm->kind == KIND_LOOPBACK) {
        // virtual ranks on one GPU: step t of rank r reads rank (r - t) mod P's shard in place (the ring's data
        // movement is the identity here; the arithmetic and the merge are the multi-GPU ones)
        for (int t = 0; t < P; ++t) {
            const std::string an = "attn" + std::to_string(t);
            pr.begin(an, sc);
            for (int r = 0; r < P; ++r) {
                const int src = ((r - t) % P + P) % P;
                AttnProblem a = ring_problem(p, q[r], k[src], v[src], parts(r) + t * p->E_loc, lses(r) + t * rows, src);
                SPA_CHECK_CUDA(launch_attention(a, sc));
                ++p->attn_launches;
            }
            pr.end(an, sc);
        }
        pr.begin("unpack", sc);   // the lse merge
        for (int r = 0; r < P; ++r) SPA_TRY(merge(r, out[r]));
        pr.end("unpack", sc);
        pr.end("total", sc);
        finish_profile(p, pr, P);
        return SPA_OK;
    }
    if (p->comm->kind == KIND_P2P) {
        // P2P ring (CUDA IPC): comm step t copies (copy engines) the block this rank holds -- its own K/V at t = 0, the
        // block received at step t-1 afterwards -- into rank r+1's receive slot t&1 and raises r+1's arrival flag t;
        // attention step t >= 1 waits for the arrival flag t-1 from rank r-1.  A slot is reused two steps later, so
        // comm step t >= 2 into rank r+1 waits for r+1's "slot free" flag t, raised once r+1's attention step t-1 and
        // its own forwarding copy of that block (comm step t-1) are done.
        SPA_TRY(ensure_stream(p->comm));
        cudaStream_t sm = p->comm->stream;
        cudaEvent_t *ev = p->sync_ev.data();
        cudaEvent_t ev_entry = ev[0], ev_done = ev[1];
        cudaEvent_t *comp = ev + 4, *cev = ev + 4 + P;
        const int r = p->comm->rank, next = (r + 1) % P, prev = (r + P - 1) % P;
        const size_t blk = (size_t)p->E_loc * 2;
        auto slotK = [&](int rank, int s) { return resolve(x, rank, BUF_WS, p->off_kvbuf + (long long)(2 * s) * blk); };
        auto slotV = [&](int rank, int s) { return resolve(x, rank, BUF_WS, p->off_kvbuf + (long long)(2 * s + 1) * blk); };
        const bool comm_on = !p->skip_comm;
        ++p->epoch;
        SPA_CHECK_CUDA(cudaEventRecord(ev_entry, sc));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(sm, ev_entry, 0));
        SPA_TRY(p2p_barrier(p, sm));   // every rank finished its previous call: its slots may be written
        for (int t = 0; t < P; ++t) {
            const void *ck = t == 0 ? k[0] : slotK(r, (t - 1) & 1);
            const void *cv = t == 0 ? v[0] : slotV(r, (t - 1) & 1);
            if (t + 1 < P) {
                const std::string cn = "in" + std::to_string(t);
                pr.begin(cn, sm);
                if (comm_on) {
                    if (t >= 1) SPA_TRY(p2p_wait_one(p, sm, FLAG_IN, t - 1, prev));   // the block to forward arrived
                    if (t >= 2) SPA_TRY(p2p_wait_one(p, sm, FLAG_OUT, t, next));      // next's slot t&1 is free
                    SPA_CHECK_CUDA(cudaMemcpyAsync(slotK(next, t & 1), ck, blk, cudaMemcpyDeviceToDevice, sm));
                    SPA_CHECK_CUDA(cudaMemcpyAsync(slotV(next, t & 1), cv, blk, cudaMemcpyDeviceToDevice, sm));
                    SPA_TRY(p2p_signal_one(p, sm, FLAG_IN, t, next));
                }
                pr.end(cn, sm);
                SPA_CHECK_CUDA(cudaEventRecord(cev[t], sm));
            }
            if (t >= 1 && comm_on) SPA_TRY(p2p_wait_one(p, sc, FLAG_IN, t - 1, prev));   // block of step t arrived
            AttnProblem a = ring_problem(p, q[0], ck, cv, parts(r) + t * p->E_loc, lses(r) + t * rows, (r - t + P) % P);
            const std::string an = "attn" + std::to_string(t);
            pr.begin(an, sc);
            SPA_CHECK_CUDA(launch_attention(a, sc));
            pr.end(an, sc);
            ++p->attn_launches;
            SPA_CHECK_CUDA(cudaEventRecord(comp[t], sc));
            // slot (t-1)&1 is free for prev's comm step t+1 once attention t and the forwarding copy t are done
            if (t >= 1 && t + 1 <= P - 2 && comm_on) {
                SPA_CHECK_CUDA(cudaStreamWaitEvent(sc, cev[t], 0));
                SPA_TRY(p2p_signal_one(p, sc, FLAG_OUT, t + 1, prev));
            }
        }
        pr.begin("unpack", sc);   // the lse merge
        SPA_TRY(merge(r, out[0]));
        pr.end("unpack", sc);
        SPA_CHECK_CUDA(cudaEventRecord(ev_done, sm));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(sc, ev_done, 0));
        pr.end("total", sc);
        finish_profile(p, pr, P);
        return SPA_OK;
    }
    // NCCL: compute on the caller's stream, K/V blocks around the ring on the comm stream
    SPA_TRY(ensure_stream(p->comm));
    cudaStream_t sm = p->comm->stream;
    cudaEvent_t *ev = p->sync_ev.data();
    cudaEvent_t ev_entry = ev[0], ev_done = ev[1];
    cudaEvent_t *comp = ev + 4, *comm = ev + 4 + P;
    const int r = p->comm->rank, next = (r + 1) % P, prev = (r + P - 1) % P;
    const size_t blk = (size_t)p->E_loc * 2;
    uint8_t *kvbuf = resolve(x, r, BUF_WS, p->off_kvbuf);
    auto slotK = [&](int s) { return kvbuf + (size_t)(2 * s) * blk; };
    auto slotV = [&](int s) { return kvbuf + (size_t)(2 * s + 1) * blk; };
    SPA_CHECK_CUDA(cudaEventRecord(ev_entry, sc));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(sm, ev_entry, 0));
    for (int t = 0; t < P; ++t) {
        const void *ck = t == 0 ? k[0] : slotK((t - 1) & 1);
        const void *cv = t == 0 ? v[0] : slotV((t - 1) & 1);
        if (t + 1 < P) {   // comm step t: pass the current block on, receive the next one
            if (t >= 1) SPA_CHECK_CUDA(cudaStreamWaitEvent(sm, comp[t - 1], 0));   // slot t%2 was read at step t-1
            const std::string cn = "in" + std::to_string(t);
            pr.begin(cn, sm);
            if (!p->skip_comm) {   // SPA_OPT_SKIP_COMM: exposed-comm measurement (slots then hold stale data)
                SPA_CHECK_NCCL(ncclGroupStart());
                SPA_CHECK_NCCL(ncclSend(ck, blk, ncclUint8, next, p->comm->nccl, sm));
                SPA_CHECK_NCCL(ncclSend(cv, blk, ncclUint8, next, p->comm->nccl, sm));
                SPA_CHECK_NCCL(ncclRecv(slotK(t & 1), blk, ncclUint8, prev, p->comm->nccl, sm));
                SPA_CHECK_NCCL(ncclRecv(slotV(t & 1), blk, ncclUint8, prev, p->comm->nccl, sm));
                SPA_CHECK_NCCL(ncclGroupEnd());
            }
            pr.end(cn, sm);
            SPA_CHECK_CUDA(cudaEventRecord(comm[t], sm));
        }
        if (t >= 1) SPA_CHECK_CUDA(cudaStreamWaitEvent(sc, comm[t - 1], 0));
        AttnProblem a = ring_problem(p, q[0], ck, cv, parts(r) + t * p->E_loc, lses(r) + t * rows, (r - t + P) % P);
        const std::string an = "attn" + std::to_string(t);
        pr.begin(an, sc);
        SPA_CHECK_CUDA(launch_attention(a, sc));
        pr.end(an, sc);
        ++p->attn_launches;
        SPA_CHECK_CUDA(cudaEventRecord(comp[t], sc));
    }
    pr.begin("unpack", sc);   // the lse merge
    SPA_TRY(merge(r, out[0]));
    pr.end("unpack", sc);
    SPA_CHECK_CUDA(cudaEventRecord(ev_done, sm));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(sc, ev_done, 0));
    pr.end("total", sc);
    finish_profile(p, pr, P);
    return SPA_OK;
}

static spa_status reshard_call(spa_plan *plan, int n, const void *const x[], void *const xh[], void *ws, void *stream,
                               bool local, bool to_head) {
    if (plan && plan->ring) return fail(SPA_ERR_INVALID, "ring plan: no reshard");
    Exec e{};
    SPA_TRY(prepare(plan, e, ws, stream, local));
    if (plan->Psrc != plan->P) return fail(SPA_ERR_INVALID, "reshard needs n_src == nranks");
    static thread_local Split one;
    one = make_split(plan->h, plan->S_l, 1);
    e.s = &one;
    e.has_attn = false;
    e.in_tensors = 1;
    for (int i = 0; i < n; ++i) {
        SPA_TRY(check_ptr(x[i], "x"));
        SPA_TRY(check_ptr(xh[i], "x_head"));
        e.ptr.xhead.push_back(xh[i]);
        if (to_head) e.ptr.q.push_back(x[i]);
        else e.ptr.out.push_back(const_cast<void *>(x[i]));
    }
    if (to_head) {
        e.has_out = false;
        // P2P: peers can only write into mapped workspaces -- receive into this rank's recvQ region ([B][S][h][D] for
        // one stage) and copy it to x_head locally (execute)
        e.q_recv_buf = peer_mem(plan) ? BUF_WS : BUF_XHEAD;
    } else {
        e.has_pack = false;
        e.o_send_buf = BUF_XHEAD;
    }
    return execute(e);
}

// ------------------------------------------------------------------ single GPU from / to host memory
// Head group i (g heads, G_h = gcd(stages, H) groups): H2D of its Q/K/V columns (2-D strided copies) on one
// stream, its attention on the caller's stream, D2H of its O columns on a third: group i's attention overlaps
// group i+1's H2D and group i-1's D2H (the copy engines run both directions at once).
spa_status spa_plan_host_workspace_bytes(const spa_plan *plan, size_t *bytes) {
    if (!plan || !bytes) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->P != 1 || plan->ring) return fail(SPA_ERR_INVALID, "host-buffer calls need a 1-rank, non-ring plan");
    *bytes = (size_t)4 * plan->sh.B * plan->sh.S * plan->sh.H * plan->sh.D * 2;
    return SPA_OK;
}

spa_status spa_attention_host(spa_plan *p, const void *q, const void *k, const void *v, void *o, void *ws,
                              void *stream) {
    if (!p || !q || !k || !v || !o || !ws) return fail(SPA_ERR_INVALID, "NULL argument");
    NvtxRange range("spa: attention from host buffers");
    if (p->P != 1 || p->ring || p->comm->kind != KIND_LOOPBACK)
        return fail(SPA_ERR_INVALID, "host-buffer calls need a 1-rank loopback plan");
    SPA_TRY(check_ptr(ws, "ws"));
    SPA_CHECK_CUDA(cudaSetDevice(p->comm->device));
    cudaStream_t sc = reinterpret_cast<cudaStream_t>(stream);
    SPA_TRY(ensure_stream(p->comm));
    cudaStream_t s_out = p->comm->stream;
    if (!p->s_h2d) SPA_CHECK_CUDA(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking));
    cudaStream_t s_in = p->s_h2d;
    const int B = p->sh.B, S = p->sh.S, H = p->sh.H, D = p->sh.D;
    const int G = p->split.G_h, g = H / G;   // head groups (stages = head-group count; query chunks unused)
    SPA_TRY(ensure_events(p, 4 + 2 * (size_t)G, 0));
    cudaEvent_t *ev = p->sync_ev.data();
    cudaEvent_t ev_entry = ev[0], ev_done = ev[1];
    cudaEvent_t *ev_in = ev + 4, *ev_comp = ev + 4 + G;
    p->attn_launches = 0;
    p->copy_launches = 0;
    const size_t row = (size_t)H * D * 2, grow = (size_t)g * D * 2, rows = (size_t)B * S;
    const size_t tensor = (size_t)B * S * H * D * 2, group = rows * grow;
    uint8_t *w = reinterpret_cast<uint8_t *>(ws);
    uint8_t *dX[4] = {w, w + tensor, w + 2 * tensor, w + 3 * tensor};   // Q, K, V, O: [G][B][S][g][D]
    const uint8_t *hX[3] = {reinterpret_cast<const uint8_t *>(q), reinterpret_cast<const uint8_t *>(k),
                            reinterpret_cast<const uint8_t *>(v)};
    SPA_CHECK_CUDA(cudaEventRecord(ev_entry, sc));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(s_in, ev_entry, 0));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(s_out, ev_entry, 0));
    for (int i = 0; i < G; ++i) {
        for (int t = 0; t < 3; ++t)
            SPA_CHECK_CUDA(cudaMemcpy2DAsync(dX[t] + i * group, grow, hX[t] + i * grow, row, grow, rows,
                                             cudaMemcpyHostToDevice, s_in));
        SPA_CHECK_CUDA(cudaEventRecord(ev_in[i], s_in));
    }
    for (int i = 0; i < G; ++i) {
        // group i's attention on compute stream i mod W (stage window): later groups fill earlier groups' wave tails
        cudaStream_t st;
        SPA_TRY(stage_stream(p, sc, i, &st));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(st, ev_in[i], 0));
        AttnProblem a{};
        a.q = dX[0] + i * group; a.k = dX[1] + i * group; a.v = dX[2] + i * group; a.o = dX[3] + i * group;
        a.B = B; a.Sq = a.Skv = S; a.n_heads = g; a.D = D;
        a.q_tok_stride = a.kv_tok_stride = a.o_tok_stride = (long long)g * D;
        a.q_batch_stride = a.kv_batch_stride = a.o_batch_stride = (long long)S * g * D;
        a.kv_len = p->kv_len;
        SPA_CHECK_CUDA(launch_attention(a, st));
        ++p->attn_launches;
        SPA_CHECK_CUDA(cudaEventRecord(ev_comp[i], st));
        SPA_CHECK_CUDA(cudaStreamWaitEvent(s_out, ev_comp[i], 0));
        SPA_CHECK_CUDA(cudaMemcpy2DAsync(reinterpret_cast<uint8_t *>(o) + i * grow, row, dX[3] + i * group, grow, grow,
                                         rows, cudaMemcpyDeviceToHost, s_out));
    }
    SPA_CHECK_CUDA(cudaEventRecord(ev_done, s_out));
    SPA_CHECK_CUDA(cudaStreamWaitEvent(sc, ev_done, 0));
    return SPA_OK;
}

// ------------------------------------------------------------------ SP layer from / to host buffers (e2e at any N)
static long long host_sp_staging_off(const spa_plan *p) {
    const long long per = p->ws_rank_bytes;
    return align_up(p->comm->kind == KIND_LOOPBACK ? per * p->P : per, 256);
}
static long long host_sp_tensor_bytes(const spa_plan *p) { return align_up((long long)p->sh.B * p->S_l * p->sh.H * p->sh.D * 2, 256); }

spa_status spa_plan_host_sp_workspace_bytes(const spa_plan *plan, size_t *bytes) {
    if (!plan || !bytes) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->ring) return fail(SPA_ERR_UNSUPPORTED, "host-buffer SP calls: Ulysses / PipeSP / Aco plans");
    if (plan->P == 1) return spa_plan_host_workspace_bytes(plan, bytes);
    const int nloc = plan->comm->kind == KIND_LOOPBACK ? plan->Psrc : 1;
    *bytes = (size_t)(host_sp_staging_off(plan) + 4LL * nloc * host_sp_tensor_bytes(plan));
    return SPA_OK;
}

static spa_status host_sp_call(spa_plan *p, int n, const void *const q[], const void *const k[], const void *const v[],
                               void *const out[], void *ws, void *stream, bool local) {
    if (!p) return fail(SPA_ERR_INVALID, "plan is NULL");
    if (p->ring) return fail(SPA_ERR_UNSUPPORTED, "host-buffer SP calls: Ulysses / PipeSP / Aco plans");
    if (p->P == 1) {
        if (n != 1 || !q[0] || !k[0] || !v[0] || !out[0]) return fail(SPA_ERR_INVALID, "NULL argument");
        return spa_attention_host(p, q[0], k[0], v[0], out[0], ws, stream);
    }
    Exec e{};
    SPA_TRY(prepare(p, e, ws, stream, local));
    e.s = &p->split;
    e.host = true;
    uint8_t *stage = reinterpret_cast<uint8_t *>(ws) + host_sp_staging_off(p);
    const long long T = host_sp_tensor_bytes(p);
    for (int i = 0; i < n; ++i) {
        if (!q[i] || !k[i] || !v[i] || !out[i]) return fail(SPA_ERR_INVALID, "NULL host buffer");
        e.hq.push_back(q[i]); e.hk.push_back(k[i]); e.hv.push_back(v[i]); e.hout.push_back(out[i]);
        uint8_t *d = stage + 4LL * i * T;   // device staging copies of this source's Q, K, V, O
        e.ptr.q.push_back(d); e.ptr.k.push_back(d + T); e.ptr.v.push_back(d + 2 * T); e.ptr.out.push_back(d + 3 * T);
    }
    return execute(e);
}

spa_status spa_pipesp_attention_hostbuf(spa_plan *plan, const void *q, const void *k, const void *v, void *out,
                                        void *ws, void *stream) {
    if (plan && plan->Psrc != plan->P && !is_source(plan, plan->comm->rank)) {   // Aco co-processor: no buffers
        if (q || k || v || out) return fail(SPA_ERR_INVALID, "co-processor ranks pass NULL q/k/v/out");
        return host_sp_call(plan, 0, nullptr, nullptr, nullptr, nullptr, ws, stream, false);
    }
    return host_sp_call(plan, 1, &q, &k, &v, &out, ws, stream, false);
}
spa_status spa_pipesp_attention_hostbuf_local(spa_plan *plan, const void *const q[], const void *const k[],
                                              const void *const v[], void *const out[], void *ws, void *stream) {
    if (!plan || !q || !k || !v || !out) return fail(SPA_ERR_INVALID, "NULL argument");
    return host_sp_call(plan, n_local_srcs(plan), q, k, v, out, ws, stream, true);
}

spa_status spa_ring_attention(spa_plan *plan, const void *q, const void *k, const void *v, void *out, void *ws,
                              void *stream) {
    return ring_call(plan, 1, &q, &k, &v, &out, ws, stream, false);
}
spa_status spa_ring_attention_local(spa_plan *plan, const void *const q[], const void *const k[],
                                    const void *const v[], void *const out[], void *ws, void *stream) {
    if (!plan || !q || !k || !v || !out) return fail(SPA_ERR_INVALID, "NULL argument");
    return ring_call(plan, plan->P, q, k, v, out, ws, stream, true);
}

spa_status spa_reshard_seq_to_head(spa_plan *plan, const void *x, void *x_head, void *ws, void *stream) {
    return reshard_call(plan, 1, &x, &x_head, ws, stream, false, true);
}
spa_status spa_reshard_head_to_seq(spa_plan *plan, const void *x_head, void *x, void *ws, void *stream) {
    const void *xx = x;
    void *xh = const_cast<void *>(x_head);
    return reshard_call(plan, 1, &xx, &xh, ws, stream, false, false);
}
spa_status spa_reshard_seq_to_head_local(spa_plan *plan, const void *const x[], void *const x_head[], void *ws,
                                         void *stream) {
    if (!plan || !x || !x_head) return fail(SPA_ERR_INVALID, "NULL argument");
    return reshard_call(plan, plan->P, x, x_head, ws, stream, true, true);
}
spa_status spa_reshard_head_to_seq_local(spa_plan *plan, const void *const x_head[], void *const x[], void *ws,
                                         void *stream) {
    if (!plan || !x || !x_head) return fail(SPA_ERR_INVALID, "NULL argument");
    std::vector<const void *> xx(x, x + plan->P);
    std::vector<void *> xh(plan->P);
    for (int i = 0; i < plan->P; ++i) xh[i] = const_cast<void *>(x_head[i]);
    return reshard_call(plan, plan->P, xx.data(), xh.data(), ws, stream, true, false);
}

spa_status spa_attention_fwd_masked(const void *q, const void *k, const void *v, void *o, int B, int Sq, int Skv,
                                    int n_heads, int D, long long q_tok_stride, long long q_batch_stride,
                                    long long kv_tok_stride, long long kv_batch_stride, long long o_tok_stride,
                                    long long o_batch_stride, const int32_t *kv_len, void *stream) {
    SPA_TRY(check_ptr(q, "q")); SPA_TRY(check_ptr(k, "k")); SPA_TRY(check_ptr(v, "v")); SPA_TRY(check_ptr(o, "o"));
    if (D != 64 && D != 96 && D != 128) return fail(SPA_ERR_UNSUPPORTED, "D must be 64, 96 or 128");
    if (B < 1 || Sq < 1 || Skv < 1 || n_heads < 1) return fail(SPA_ERR_SHAPE, "B, Sq, Skv, n_heads must be >= 1");
    for (long long st : {q_tok_stride, q_batch_stride, kv_tok_stride, kv_batch_stride, o_tok_stride, o_batch_stride})
        if (st % 8) return fail(SPA_ERR_INVALID, "strides must be multiples of 8 elements (16 bytes)");
    if (q_tok_stride < (long long)n_heads * D || kv_tok_stride < (long long)n_heads * D ||
        o_tok_stride < (long long)n_heads * D)
        return fail(SPA_ERR_SHAPE, "token stride smaller than n_heads*D");
    if (kv_len && reinterpret_cast<uintptr_t>(kv_len) % 4) return fail(SPA_ERR_INVALID, "kv_len not 4-byte aligned");
    AttnProblem a{q, k, v, o, B, Sq, Skv, n_heads, D, q_tok_stride, q_batch_stride,
                  kv_tok_stride, kv_batch_stride, o_tok_stride, o_batch_stride, kv_len};
    cudaError_t e = launch_attention(a, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(SPA_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
    return SPA_OK;
}

spa_status spa_attention_fwd_ex(const void *q, const void *k, const void *v, void *o, int B, int Sq, int Skv,
                                int n_heads, int D, long long q_tok_stride, long long q_batch_stride,
                                long long kv_tok_stride, long long kv_batch_stride, long long o_tok_stride,
                                long long o_batch_stride, const int32_t *kv_len, int out_fp32, float *lse,
                                void *stream) {
    SPA_TRY(check_ptr(q, "q")); SPA_TRY(check_ptr(k, "k")); SPA_TRY(check_ptr(v, "v")); SPA_TRY(check_ptr(o, "o"));
    if (D != 64 && D != 96 && D != 128) return fail(SPA_ERR_UNSUPPORTED, "D must be 64, 96 or 128");
    if (B < 1 || Sq < 1 || Skv < 1 || n_heads < 1) return fail(SPA_ERR_SHAPE, "B, Sq, Skv, n_heads must be >= 1");
    if (out_fp32 != 0 && out_fp32 != 1) return fail(SPA_ERR_INVALID, "out_fp32 must be 0 or 1");
    for (long long st : {q_tok_stride, q_batch_stride, kv_tok_stride, kv_batch_stride, o_tok_stride, o_batch_stride})
        if (st % 8) return fail(SPA_ERR_INVALID, "strides must be multiples of 8 elements (16 bytes)");
    if (q_tok_stride < (long long)n_heads * D || kv_tok_stride < (long long)n_heads * D ||
        o_tok_stride < (long long)n_heads * D)
        return fail(SPA_ERR_SHAPE, "token stride smaller than n_heads*D");
    if (kv_len && reinterpret_cast<uintptr_t>(kv_len) % 4) return fail(SPA_ERR_INVALID, "kv_len not 4-byte aligned");
    if (lse && reinterpret_cast<uintptr_t>(lse) % 4) return fail(SPA_ERR_INVALID, "lse not 4-byte aligned");
    AttnProblem a{q, k, v, out_fp32 ? nullptr : o, B, Sq, Skv, n_heads, D, q_tok_stride, q_batch_stride,
                  kv_tok_stride, kv_batch_stride, o_tok_stride, o_batch_stride, kv_len};
    if (out_fp32) a.o32 = o;
    a.lse = lse;
    cudaError_t e = launch_attention(a, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(SPA_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
    return SPA_OK;
}

spa_status spa_attention_fwd(const void *q, const void *k, const void *v, void *o, int B, int Sq, int Skv,
                             int n_heads, int D, long long q_tok_stride, long long q_batch_stride,
                             long long kv_tok_stride, long long kv_batch_stride, long long o_tok_stride,
                             long long o_batch_stride, void *stream) {
    return spa_attention_fwd_masked(q, k, v, o, B, Sq, Skv, n_heads, D, q_tok_stride, q_batch_stride, kv_tok_stride,
                                    kv_batch_stride, o_tok_stride, o_batch_stride, nullptr, stream);
}

// ------------------------------------------------------------------ describe (host only)
spa_status spa_plan_describe_pack(const spa_plan *plan, int rank, spa_copy_desc *out, int max, int *n) {
    if (!plan || !n) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->ring) return fail(SPA_ERR_INVALID, "ring plan: nothing to describe");
    *n = 0;
    if (plan->P == 1 || !is_source(plan, rank)) return SPA_OK;
    const long long offs[3] = {plan->off_sendQ, plan->off_sendK, plan->off_sendV};
    for (int t = 0; t < 3; ++t) {
        std::vector<CopyJob> jobs;
        pack_jobs(plan, plan->split, rank, nullptr, 0, nullptr, jobs);
        for (const CopyJob &j : jobs) {
            if (*n >= max) return fail(SPA_ERR_INVALID, "describe: output too small");
            // job pointers are offsets from NULL here: source offset into the user buffer, destination into ws
            out[(*n)++] = to_desc(j, BUF_Q + t, rank, (long long)reinterpret_cast<uintptr_t>(j.src), BUF_WS, rank,
                                  offs[t] + (long long)reinterpret_cast<uintptr_t>(j.dst));
        }
    }
    return SPA_OK;
}

spa_status spa_plan_describe_unpack(const spa_plan *plan, int rank, spa_copy_desc *out, int max, int *n) {
    if (!plan || !n) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->ring) return fail(SPA_ERR_INVALID, "ring plan: nothing to describe");
    *n = 0;
    if (plan->P == 1 || !is_source(plan, rank)) return SPA_OK;
    std::vector<CopyJob> jobs;
    unpack_jobs(plan, plan->split, rank, nullptr, 0, nullptr, jobs);
    for (const CopyJob &j : jobs) {
        if (*n >= max) return fail(SPA_ERR_INVALID, "describe: output too small");
        out[(*n)++] = to_desc(j, BUF_WS, rank, plan->off_orecv + (long long)reinterpret_cast<uintptr_t>(j.src),
                              BUF_OUT, rank, (long long)reinterpret_cast<uintptr_t>(j.dst));
    }
    return SPA_OK;
}

spa_status spa_plan_describe_messages(const spa_plan *plan, int stage, int dir, int rank, spa_msg *out, int max,
                                      int *n) {
    if (!plan || !n) return fail(SPA_ERR_INVALID, "NULL argument");
    if (plan->ring) return fail(SPA_ERR_INVALID, "ring plan: nothing to describe");
    if (stage < 0 || stage >= plan->split.n() || rank < 0 || rank >= plan->P)
        return fail(SPA_ERR_INVALID, "bad stage/rank");
    std::vector<Msg> m;
    if (plan->P > 1) {
        if (dir == 0) gen_in_msgs(plan, plan->split, stage, rank, 7, BUF_WS, m);
        else gen_out_msgs(plan, plan->split, stage, rank, BUF_WS, m);
    }
    if ((int)m.size() > max) return fail(SPA_ERR_INVALID, "describe: output too small");
    for (size_t i = 0; i < m.size(); ++i) out[i] = {m[i].peer, m[i].is_recv, m[i].buf, m[i].off, m[i].bytes};
    *n = (int)m.size();
    return SPA_OK;
}

// Ring step t of `rank` in the order ring_call issues it: send K, send V (the block held: the caller's at t = 0, else
// receive slot (t-1)&1) to rank+1, receive K, V from rank-1 into slot t&1.  USP plans: the ring sub-plan's step with
// peers as global ranks (ring of u = rank % U: ranks rho*U + u).
spa_status spa_plan_describe_ring(const spa_plan *p, int step, int rank, spa_msg *out, int max, int *n) {
    if (!p || !n || (!out && max > 0)) return fail(SPA_ERR_INVALID, "NULL argument");
    if (!p->ring) return fail(SPA_ERR_INVALID, "not a ring plan");
    if (rank < 0 || rank >= p->P) return fail(SPA_ERR_INVALID, "bad rank");
    *n = 0;
    if (p->U > 1) {
        const int U = p->U, u = rank % U;
        SPA_TRY(spa_plan_describe_ring(p->ring_plan, step, rank / U, out, max, n));
        for (int i = 0; i < *n; ++i) out[i].peer = out[i].peer * U + u;
        return SPA_OK;
    }
    const int P = p->P;
    if (step < 0 || step >= std::max(1, P - 1)) return fail(SPA_ERR_INVALID, "bad ring step");
    if (P == 1) return SPA_OK;
    if (max < 4) return fail(SPA_ERR_INVALID, "describe: output too small");
    const long long blk = p->E_loc * 2;
    const int next = (rank + 1) % P, prev = (rank + P - 1) % P;
    const int cur = (step - 1) & 1, nxt = step & 1;
    out[0] = {next, 0, step == 0 ? BUF_K : BUF_WS, step == 0 ? 0 : p->off_kvbuf + (2LL * cur) * blk, blk};
    out[1] = {next, 0, step == 0 ? BUF_V : BUF_WS, step == 0 ? 0 : p->off_kvbuf + (2LL * cur + 1) * blk, blk};
    out[2] = {prev, 1, BUF_WS, p->off_kvbuf + (2LL * nxt) * blk, blk};
    out[3] = {prev, 1, BUF_WS, p->off_kvbuf + (2LL * nxt + 1) * blk, blk};
    *n = 4;
    return SPA_OK;
}

spa_status spa_plan_describe_attention(const spa_plan *p, int stage, int rank, spa_attn_desc *out) {
    if (!p || !out) return fail(SPA_ERR_INVALID, "NULL argument");
    if (p->ring) return fail(SPA_ERR_INVALID, "ring plan: nothing to describe");
    if (stage < 0 || stage >= p->split.n() || rank < 0 || rank >= p->P) return fail(SPA_ERR_INVALID, "bad stage/rank");
    const Split &s = p->split;
    const int kh = stage / s.C, c = stage % s.C;
    const long long Lst = Lstage(p, s, c);
    out->q_off = p->off_recvQ + base_stage(p, s, kh, c) * 2;
    out->k_off = p->off_recvK + idx_kv(p, s, kh, 0, 0) * 2;
    out->v_off = p->off_recvV + idx_kv(p, s, kh, 0, 0) * 2;
    out->o_off = p->off_O + base_stage(p, s, kh, c) * 2;
    out->B = p->sh.B; out->Sq = (int)Lst; out->Skv = p->sh.S; out->n_heads = real_heads(p, s, rank, kh);
    out->q_tok_stride = out->kv_tok_stride = (long long)s.g * p->sh.D;
    out->q_batch_stride = Lst * s.g * p->sh.D;
    out->kv_batch_stride = (long long)p->sh.S * s.g * p->sh.D;
    return SPA_OK;
}

}  // extern "C"
