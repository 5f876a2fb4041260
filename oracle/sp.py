"""Sequence-parallel path simulated over P virtual ranks (TEST INFRASTRUCTURE ONLY).

Every step is an explicit index permutation over numpy arrays (any dtype: the
bf16 bit patterns as uint16 for bit-exact reshard checks, float64 for the
attention result).  Attention itself is injected as ``attn(q_rows, K, V)`` so the
same per-row routine (oracle.attention_rows) serves the sharded and unsharded
evaluations -- which is why the fp64 SP result is bit-identical to unsharded
attention (reading R8).

Paper passages followed, in the paper's order:
  * seq->head all-to-all of Q, K, V        PAPER.md:65-67 (§2 "Sequence parallelism"), :29
  * Alg. 1 loop: attention(j) -> All_to_All(results[j]) -> append chunks
  * concat + view(-1,h,n,D) + permute(0,2,1,3) + view(-1,h*n,D)
  * index maps k_orig(i,j)=i*h+j, k_mod(i,j)=j*n+i and Psi=phi^-1 pi phi
  * Aco: intra-group All-to-All, then P2P to the Decoding GPUs, attention in
    both groups, results back by P2P + intra-group All-to-All
  * head padding

Readings: n = P ranks, h = H/P (R3); contiguous head blocks
per rank (R4); source-rank-major chunk order (R5); head groups of g heads and
query chunks give N_st = G_h*C stages with Psi_g (R6, R7).
"""
from __future__ import annotations

import math
from typing import Callable, List, Sequence, Tuple

import numpy as np

Attn = Callable[[np.ndarray, np.ndarray, np.ndarray], np.ndarray]


# ---------------------------------------------------------------- primitives
def shard_bounds(S: int, P: int) -> List[int]:
    """Token bounds of P sequence shards that differ in length by at most one (R9; the SPEC's
    ShardedTensor "differ by <= 1"): the first S % P ranks hold one token more."""
    base, extra = divmod(S, P)
    b = [0]
    for r in range(P):
        b.append(b[-1] + base + (1 if r < extra else 0))
    return b


def shard_seq(X: np.ndarray, P: int, uneven: bool = False) -> List[np.ndarray]:
    """X [B,S,H,D] -> P sequence shards (rank r holds tokens [bounds[r], bounds[r+1])); equal shards of S/P
    tokens unless uneven=True allows S % P != 0."""
    B, S, H, D = X.shape
    if S % P and not uneven:
        raise ValueError("S % P != 0")
    b = shard_bounds(S, P)
    return [X[:, b[r]:b[r + 1]].copy() for r in range(P)]


def all_to_all(send: Sequence[Sequence[np.ndarray]]) -> List[List[np.ndarray]]:
    """send[p][q] = chunk rank p sends to rank q.  Returns recv[q][p] (source-rank order)."""
    n = len(send)
    for p in range(n):
        if len(send[p]) != n:
            raise ValueError("each rank must provide one chunk per destination")
    return [[send[p][q] for p in range(n)] for q in range(n)]


def seq_to_head(shards: Sequence[np.ndarray]) -> List[np.ndarray]:
    """Ulysses input all-to-all: R_r[b, p*S_l+t, j] = X_p[b, t, r*h+j]."""
    P = len(shards)
    B, S_l, H, D = shards[0].shape
    if H % P:
        raise ValueError("H % P != 0")
    h = H // P
    send = [[x[:, :, q * h:(q + 1) * h] for q in range(P)] for x in shards]
    recv = all_to_all(send)
    return [np.concatenate(recv[r], axis=1) for r in range(P)]


def head_to_seq(heads: Sequence[np.ndarray], bounds: Sequence[int] = None) -> List[np.ndarray]:
    """Ulysses output all-to-all (one exchange after all heads):
    out_q[b, t, r*h+j] = R_r[b, bounds[q]+t, j] (bounds: the sequence shards, equal by default)."""
    P = len(heads)
    B, S, h, D = heads[0].shape
    if bounds is None:
        bounds = shard_bounds(S, P)
    send = [[y[:, bounds[q]:bounds[q + 1]] for q in range(P)] for y in heads]
    recv = all_to_all(send)
    return [np.concatenate(recv[q], axis=2) for q in range(P)]


def k_orig(i: int, j: int, h: int) -> int:
    """head held by GPU i as local head j in the original (Ulysses) order."""
    return i * h + j


def k_mod(i: int, j: int, n: int) -> int:
    """position of that head after PipeSP's per-head all-to-alls."""
    return j * n + i


def psi(T: np.ndarray, h: int, n: int) -> np.ndarray:
    """The paper's fix: view(-1,h,n,D) -> permute(0,2,1,3) -> view(-1,h*n,D).
    T has the head axis second-to-last: [..., h*n, D]."""
    lead = T.shape[:-2]
    D = T.shape[-1]
    t = T.reshape((-1, h, n, D))
    t = np.transpose(t, (0, 2, 1, 3))
    return np.ascontiguousarray(t).reshape(lead + (h * n, D))


def psi_g(T: np.ndarray, G_h: int, P: int, g: int) -> np.ndarray:
    """Psi generalised to head groups of g heads (R6):
    view(-1,G_h,P,g,D) -> permute(0,2,1,3,4) -> view(-1,H,D).  g=1 is the paper's Psi."""
    lead = T.shape[:-2]
    D = T.shape[-1]
    t = T.reshape((-1, G_h, P, g, D))
    t = np.transpose(t, (0, 2, 1, 3, 4))
    return np.ascontiguousarray(t).reshape(lead + (G_h * P * g, D))


def stage_split(h: int, n_stages: int) -> Tuple[int, int, int]:
    """N_st = G_h * C (R7): G_h = gcd(N_st, h) head groups of g = h/G_h heads,
    C = N_st/G_h query chunks per head group."""
    if n_stages < 1:
        raise ValueError("stages < 1")
    G_h = math.gcd(n_stages, h)
    return G_h, n_stages // G_h, h // G_h


def chunk_bounds(S_l: int, C: int) -> List[Tuple[int, int]]:
    """Query chunk c of every source rank's local tokens: [c*S_l//C, (c+1)*S_l//C) (extents differ by <=1)."""
    if C > S_l:
        raise ValueError("more query chunks than local tokens")
    return [(c * S_l // C, (c + 1) * S_l // C) for c in range(C)]


def pad_heads(H: int, n: int) -> Tuple[int, int]:
    """Smallest multiple of n that is >= H, and the pad count."""
    if H < 1 or n < 1:
        raise ValueError("H, n >= 1")
    Hp = -(-H // n) * n
    return Hp, Hp - H


def padded_forward(Qs, Ks, Vs, n_owners: int, forward) -> List[np.ndarray]:
    """Head padding ("padding increases the head count to 28 so that each GPU
    handles 4 heads"): append pad_heads(H, n_owners)[1] all-zero heads to every shard's Q, K, V, run
    `forward(Qs', Ks', Vs')` (e.g. ulysses_forward / pipesp_forward) on the padded problem, and drop
    the pad heads from every output shard.  Heads are independent, so the real heads'
    result is the unpadded one; a zero pad head attends with uniform weights to zero values -> 0."""
    B, S_l, H, D = Qs[0].shape
    Hp, n_pad = pad_heads(H, n_owners)
    if n_pad == 0:
        return forward(Qs, Ks, Vs)
    padz = np.zeros((B, S_l, n_pad, D), dtype=np.float64)
    pad = lambda xs: [np.concatenate([x, padz], axis=2) for x in xs]  # noqa: E731
    outs = forward(pad(Qs), pad(Ks), pad(Vs))
    return [np.ascontiguousarray(o[:, :, :H]) for o in outs]


# ---------------------------------------------------------------- Ring attention (USP fallback)
def lse_merge(parts, lses):
    """Combine softmax-normalised partial results over disjoint key blocks (R21):
    O = sum_i exp(lse_i - M) O_i / sum_i exp(lse_i - M), M = max_i lse_i; lse = M + ln sum_i exp(lse_i - M).
    parts[i]: [..., D], lses[i]: [...] (float64).  Rows with every lse = -inf give 0 and lse -inf."""
    L = np.stack(lses)                      # [n, ...]
    M = L.max(axis=0)
    finite = np.isfinite(M)
    Ms = np.where(finite, M, 0.0)
    W = np.where(np.isfinite(L), np.exp(L - Ms), 0.0)
    den = W.sum(axis=0)
    num = sum(W[i][..., None] * parts[i] for i in range(len(parts)))
    out = np.where(finite[..., None], num / np.where(finite, den, 1.0)[..., None], 0.0)
    lse = np.where(finite, Ms + np.log(np.where(finite, den, 1.0)), -np.inf)
    return out, lse


def ring_forward(Qs, Ks, Vs, attn_lse) -> List[np.ndarray]:
    """Ring attention over P ranks (the paper's Ring-Attention fallback when H is not divisible, PAPER.md:171;
    it gives no procedure -- DESIGN.md R21): rank r keeps its query shard and all heads; at step t it attends
    to the K/V shard of rank (r - t) mod P (the shards travel around the ring r -> r+1), giving a partial
    result and its lse per row; the P partials are combined with lse_merge.  attn_lse(q [R,D], K, V) ->
    (O [R,D], lse [R]).  No head divisibility is needed."""
    P = len(Qs)
    B, S_l, H, D = Qs[0].shape
    outs = []
    for r in range(P):
        parts, lses = [], []
        for t in range(P):
            src = (r - t) % P
            O = np.empty((B, S_l, H, D))
            L = np.empty((B, S_l, H))
            for b in range(B):
                for k in range(H):
                    O[b, :, k], L[b, :, k] = attn_lse(np.ascontiguousarray(Qs[r][b, :, k]),
                                                      np.ascontiguousarray(Ks[src][b, :, k]),
                                                      np.ascontiguousarray(Vs[src][b, :, k]))
            parts.append(O)
            lses.append(L)
        outs.append(lse_merge(parts, lses)[0])
    return outs


def usp_forward(Qs, Ks, Vs, U: int, attn_lse) -> List[np.ndarray]:
    """USP hybrid (PAPER.md:171 -- Ulysses degree U x Ring degree R = P/U; R21): ranks
    [rho*U, rho*U+U) form Ulysses group rho.  1. seq->head all-to-all inside each group; 2. ring attention over
    the R groups among the ranks with the same position u in their group (heads u*H/U.. of every group's
    tokens); 3. head->seq all-to-all inside each group."""
    P = len(Qs)
    R = P // U
    heads = [None] * P
    for t, X in enumerate((Qs, Ks, Vs)):
        for rho in range(R):
            hs = seq_to_head(X[rho * U:(rho + 1) * U])            # step 1, group rho
            for u in range(U):
                if heads[rho * U + u] is None:
                    heads[rho * U + u] = [None, None, None]
                heads[rho * U + u][t] = hs[u]
    O = [None] * P
    for u in range(U):                                          # step 2, ring of position u
        members = [rho * U + u for rho in range(R)]
        outs = ring_forward([heads[i][0] for i in members], [heads[i][1] for i in members],
                            [heads[i][2] for i in members], attn_lse)
        for rho, i in enumerate(members):
            O[i] = outs[rho]
    res = []
    for rho in range(R):                                        # step 3
        res.extend(head_to_seq(O[rho * U:(rho + 1) * U]))
    return res


# ---------------------------------------------------------------- attention per rank
def _attn_heads(Rq: np.ndarray, Rk: np.ndarray, Rv: np.ndarray, rows: np.ndarray, heads: Sequence[int],
                attn: Attn) -> np.ndarray:
    """attention for the given query rows of the given local heads on one rank -> [B, len(rows), len(heads), D]."""
    B, S, h, D = Rq.shape
    out = np.empty((B, len(rows), len(heads), D), dtype=np.float64)
    for b in range(B):
        for jj, j in enumerate(heads):
            out[b, :, jj, :] = attn(np.ascontiguousarray(Rq[b, rows, j, :]),
                                    np.ascontiguousarray(Rk[b, :, j, :]),
                                    np.ascontiguousarray(Rv[b, :, j, :]))
    return out


# ---------------------------------------------------------------- Ulysses / PipeSP
def ulysses_forward(Qs, Ks, Vs, attn: Attn) -> List[np.ndarray]:
    """Fig. 3(a): 3 all-to-alls, attention on all local heads, 1 all-to-all."""
    Rq, Rk, Rv = seq_to_head(Qs), seq_to_head(Ks), seq_to_head(Vs)
    P = len(Qs)
    B, S, h, D = Rq[0].shape
    O = [_attn_heads(Rq[r], Rk[r], Rv[r], np.arange(S), range(h), attn) for r in range(P)]
    return head_to_seq(O)


def pipesp_forward(Qs, Ks, Vs, n_stages: int, attn: Attn, return_tmod: bool = False):
    """Alg. 1 generalised to N_st = G_h*C stages (R6/R7).

    Stage k = (head group kh, query chunk c).  Per stage: attention of local heads
    kh*g..kh*g+g-1 for the query rows of chunk c of every source block, then the
    stage's all-to-all: dest q receives from src r the rows [q*S_l+c0, q*S_l+c1) of
    those heads, appended to its chunk list (Alg. 1 l.7-8).  After the loop: per
    query chunk, concat along heads (l.10) -> T^mod with head position
    kh*P*g + r*g + jj; Psi_g (l.11-13) restores k_orig = r*h + kh*g + jj.
    With g=1, C=1 this is exactly the paper's per-head loop and Psi.
    """
    P = len(Qs)
    B, _, H, D = Qs[0].shape
    h = H // P
    lens = [x.shape[1] for x in Qs]                 # sequence shards may differ by one token (R9)
    starts = np.concatenate([[0], np.cumsum(lens)]).astype(int)
    G_h, C, g = stage_split(h, n_stages)
    cbs = [chunk_bounds(n, C) for n in lens]        # query chunk c of source p: its local [c0_p, c1_p)
    Rq, Rk, Rv = seq_to_head(Qs), seq_to_head(Ks), seq_to_head(Vs)  # leading all-to-alls
    chunks = [[[] for _ in range(C)] for _ in range(P)]  # chunks[dest][c] = list of stage pieces
    for kh in range(G_h):
        heads = list(range(kh * g, (kh + 1) * g))
        for c in range(C):
            # rows of chunk c from every source block p: starts[p] + [c0_p, c1_p)
            rows = np.concatenate([np.arange(starts[p] + cbs[p][c][0], starts[p] + cbs[p][c][1]) for p in range(P)])
            results = [_attn_heads(Rq[r], Rk[r], Rv[r], rows, heads, attn) for r in range(P)]
            offs = np.concatenate([[0], np.cumsum([cbs[q][c][1] - cbs[q][c][0] for q in range(P)])]).astype(int)
            send = [[results[r][:, offs[q]:offs[q + 1]] for q in range(P)] for r in range(P)]
            recv = all_to_all(send)                      # the stage's All_to_All (Alg. 1 l.7)
            for q in range(P):
                # pieces from src r: [B, L, g, D]; stage piece = concat over r along heads -> [B,L,P*g,D]
                chunks[q][c].append(np.concatenate(recv[q], axis=2))
    outs, tmods = [], []
    for q in range(P):
        per_chunk = []
        tm = []
        for c in range(C):
            Tmod = np.concatenate(chunks[q][c], axis=2)  # concat(chunks, dim=heads) (Alg. 1 l.10)
            tm.append(Tmod)
            per_chunk.append(psi_g(Tmod, G_h, P, g))
        outs.append(np.concatenate(per_chunk, axis=1))
        tmods.append(np.concatenate(tm, axis=1))
    return (outs, tmods) if return_tmod else outs


# ---------------------------------------------------------------- Aco relay
def aco_forward(Qs, Ks, Vs, n_decode: int, attn: Attn) -> List[np.ndarray]:
    """Aco prompt-1 stage as the paper describes it (Fig. 4):

    1. Denoising GPUs (len(Qs) = N_d) run the intra-group seq->head All-to-All:
       denoise rank r holds heads [r*h_d, (r+1)*h_d), full sequence.
    2. Each denoise rank keeps its first h = H/N heads and ships the remaining
       h_d - h heads (Q, K, V) point-to-point to the Decoding GPUs, filled in
       (rank, head) order, h heads per decoding GPU.
    3. Both groups run attention on their heads.
    4. Decoding GPUs return results by P2P; denoise ranks run the intra-group
       head->seq All-to-All and obtain full-head, partial-sequence outputs.
    Requires H % N_d == 0 and H % N == 0 (no padding).
    """
    N_d = len(Qs)
    B, S_l, H, D = Qs[0].shape
    N = N_d + n_decode
    if H % N_d or H % N:
        raise ValueError("Aco relay needs H divisible by N_denoise and by N")
    h_d, h = H // N_d, H // N
    Rq, Rk, Rv = seq_to_head(Qs), seq_to_head(Ks), seq_to_head(Vs)      # step 1
    S = Rq[0].shape[1]
    shipped = [(r, j) for r in range(N_d) for j in range(h, h_d)]       # step 2
    assert len(shipped) == n_decode * h
    O = [np.empty((B, S, h_d, D)) for _ in range(N_d)]
    for r in range(N_d):                                                 # step 3, denoise group
        O[r][:, :, :h] = _attn_heads(Rq[r], Rk[r], Rv[r], np.arange(S), range(h), attn)
    for dec in range(n_decode):                                          # step 3, decoding group
        mine = shipped[dec * h:(dec + 1) * h]
        q = np.stack([Rq[r][:, :, j] for r, j in mine], axis=2)         # received by P2P
        k = np.stack([Rk[r][:, :, j] for r, j in mine], axis=2)
        v = np.stack([Rv[r][:, :, j] for r, j in mine], axis=2)
        res = _attn_heads(q, k, v, np.arange(S), range(h), attn)
        for jj, (r, j) in enumerate(mine):                               # step 4, P2P back
            O[r][:, :, j] = res[:, :, jj]
    return head_to_seq(O)                                                # step 4, intra-group a2a


# ---------------------------------------------------------------- Aco performance model
def aco_times(t_L: float, t_A: float, n_denoise: int, n_total: int) -> Tuple[float, float]:
    """Eqs. (1)-(2): T_baseline = t_L + t_A; T_coop = t_L + t_A * N_denoise / N."""
    return t_L + t_A, t_L + t_A * n_denoise / n_total


def aco_ideal_speedup(t_L: float, t_A: float, n_denoise: int, n_total: int) -> float:
    """Eq. (3): S = T_baseline / T_coop."""
    base, coop = aco_times(t_L, t_A, n_denoise, n_total)
    return base / coop
