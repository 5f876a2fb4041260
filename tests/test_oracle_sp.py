"""Pins for the sequence-parallel simulation in oracle/sp.py (CPU only).

Independent anchors: SPEC hand cases (all_to_all n=2, layout_fix n=2,h=2, pre-fix
order [0,2,1,3]), the paper's index maps k_orig / k_mod,
label tracing (every element carries its own (token, head) label, attention
replaced by the identity), conservation, and fp64 SP == unsharded attention."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from oracle import sp


def _golden(golden_dir):
    with open(os.path.join(golden_dir, "layout_fix_cases.json")) as f:
        return json.load(f)


# ----------------------------------------------------------- all_to_all
def test_all_to_all_hand_case_and_identity(golden_dir):
    g = _golden(golden_dir)
    recv = sp.all_to_all(g["a2a_in"])
    assert [list(r) for r in recv] == g["a2a_out"]
    assert sp.all_to_all([["x"]]) == [["x"]]                # n=1 identity


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_seq_head_roundtrip_and_conservation(P):
    rng = np.random.default_rng(P)
    B, S, H, D = 2, 8 * P, 2 * P, 3
    X = rng.integers(0, 1 << 16, size=(B, S, H, D)).astype(np.uint16)
    shards = sp.shard_seq(X, P)
    heads = sp.seq_to_head(shards)
    back = sp.head_to_seq(heads)                            # SPEC.md:123 round trip
    for r in range(P):
        assert np.array_equal(back[r], shards[r])
    allv = np.sort(np.concatenate([h.ravel() for h in heads]))
    assert np.array_equal(allv, np.sort(X.ravel()))         # SPEC.md:174 multiset conservation
    if P == 1:
        assert np.array_equal(heads[0], X)                   # P=1 is the identity reshard


def test_seq_to_head_labels():
    """R_r[b, s, j] must hold global token s, global head r*h+j (contiguous head blocks)."""
    P, B, S, H, D = 4, 2, 16, 8, 1
    tok = np.arange(S)[None, :, None, None]
    head = np.arange(H)[None, None, :, None]
    X = (np.zeros((B, S, H, D)) + tok * 1000 + head + 1e6 * np.arange(B)[:, None, None, None])
    heads = sp.seq_to_head(sp.shard_seq(X, P))
    h = H // P
    for r in range(P):
        for b, s, j in itertools.product(range(B), range(S), range(h)):
            assert heads[r][b, s, j, 0] == b * 1e6 + s * 1000 + r * h + j


# ----------------------------------------------------------- Psi
def test_layout_fix_hand_case(golden_dir):
    g = _golden(golden_dir)
    labels = {c: i for i, c in enumerate("ABCD")}
    T = np.array([labels[c] for c in g["layout_fix_in"]], dtype=np.float64).reshape(1, 4, 1)
    out = sp.psi(T, h=2, n=2)
    assert ["ABCD"[int(v)] for v in out.ravel()] == g["layout_fix_out"]


def test_prefix_order_n2_h2(golden_dir):
    """Before the fix, PipeSP's head order is [0,2,1,3]."""
    g = _golden(golden_dir)
    P, H, S = 2, 4, 4
    X = np.zeros((1, S, H, 1)) + np.arange(H)[None, None, :, None]
    shards = sp.shard_seq(X, P)
    ident = lambda q, K, V: q  # noqa: E731  label routing only
    outs, tmods = sp.pipesp_forward(shards, shards, shards, n_stages=2, attn=ident, return_tmod=True)
    for q in range(P):
        assert list(tmods[q][0, 0, :, 0].astype(int)) == g["prefix_order_n2_h2"]
        assert list(outs[q][0, 0, :, 0].astype(int)) == [0, 1, 2, 3]


@pytest.mark.parametrize("n,h", list(itertools.product(range(1, 9), range(1, 9))))
def test_psi_exhaustive_against_index_maps(n, h):
    """Psi T^mod = T^orig for label tensors built from k_orig/k_mod."""
    H = n * h
    Tmod = np.empty((1, H, 1))
    for i in range(n):
        for j in range(h):
            Tmod[0, j * n + i, 0] = i * h + j          # position k_mod(i,j) holds head k_orig(i,j)
    out = sp.psi(Tmod, h=h, n=n)
    assert np.array_equal(out[0, :, 0], np.arange(H))
    assert sp.k_mod(1 % n, 0, n) == 1 % n and sp.k_orig(1 % n, 0, h) == (1 % n) * h
    if n == 1 or h == 1:
        assert np.array_equal(out, Tmod)


# ----------------------------------------------------------- label routing through the full path
def _labelled(B, S, H, D):
    b = np.arange(B)[:, None, None, None]
    s = np.arange(S)[None, :, None, None]
    k = np.arange(H)[None, None, :, None]
    d = np.arange(D)[None, None, None, :]
    return (b * 10_000_000 + s * 10_000 + k * 100 + d).astype(np.float64)


def _stage_cfgs(h):
    return sorted({1, 2, 3, 4, 6, 8, 12, 24, h, 2 * h} | set(range(1, h + 1)))


@pytest.mark.parametrize("P,H", [(1, 4), (2, 4), (2, 6), (4, 8), (4, 12), (8, 24), (3, 6)])
def test_pipesp_routes_every_element_home(P, H):
    """Identity attention: output == input for every stage config (head groups g | h, query chunks)."""
    B, S, D = 2, 8 * P, 2
    X = _labelled(B, S, H, D)
    shards = sp.shard_seq(X, P)
    ident = lambda q, K, V: q  # noqa: E731
    h = H // P
    for n_st in _stage_cfgs(h):
        G_h, C, g = sp.stage_split(h, n_st)
        if C > S // P:
            continue
        outs = sp.pipesp_forward(shards, shards, shards, n_st, ident)
        for r in range(P):
            assert np.array_equal(outs[r], shards[r]), (P, H, n_st)


def test_stage_split_and_chunks():
    assert sp.stage_split(3, 24) == (3, 8, 1)
    assert sp.stage_split(3, 4) == (1, 4, 3)
    assert sp.stage_split(3, 1) == (1, 1, 3)
    assert sp.stage_split(24, 24) == (24, 1, 1)
    assert sp.stage_split(24, 16) == (8, 2, 3)
    b = sp.chunk_bounds(14850, 8)
    assert b[0][0] == 0 and b[-1][1] == 14850
    sizes = {e - s for s, e in b}
    assert max(sizes) - min(sizes) <= 1 and sum(e - s for s, e in b) == 14850


# ----------------------------------------------------------- SP == unsharded (fp64, bit-exact)
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_sp_equals_unsharded_bit_exact(P):
    rng = np.random.default_rng(100 + P)
    B, S, H, D = 1, 4 * P, 8, 4
    Q, K, V = (rng.standard_normal((B, S, H, D)) for _ in range(3))
    ref = oracle.mha_unsharded(Q, K, V, nthreads=1)
    attn = lambda q, k, v: oracle.attention_rows(q, k, v, nthreads=1)  # noqa: E731
    h = H // P
    Qs, Ks, Vs = sp.shard_seq(Q, P), sp.shard_seq(K, P), sp.shard_seq(V, P)
    for n_st in sorted({1, h, 2 * h, 2}):
        outs = sp.pipesp_forward(Qs, Ks, Vs, n_st, attn)
        assert np.array_equal(np.concatenate(outs, axis=1), ref), n_st
    assert np.array_equal(np.concatenate(sp.ulysses_forward(Qs, Ks, Vs, attn), axis=1), ref)


def test_pipesp_equals_ulysses_seeded_sweep():
    """SPEC.md:379 acceptance #2: >=100 seeded cases, n in {1,2,4}, H in {4,8,16}, S in {8,16,32},
    B in {1,2}, D in {4,8}, 0 ulp (the paper's per-head loop, N_st = h)."""
    attn = lambda q, k, v: oracle.attention_rows(q, k, v, nthreads=1)  # noqa: E731
    cases = list(itertools.product([1, 2, 4], [4, 8, 16], [8, 16, 32], [1, 2], [4, 8]))
    rng = np.random.default_rng(2024)
    picked = [cases[i] for i in rng.choice(len(cases), size=100, replace=False)]
    for seed, (n, H, S, B, D) in enumerate(picked):
        r = np.random.default_rng(seed)
        Q, K, V = (r.standard_normal((B, S, H, D)) for _ in range(3))
        Qs, Ks, Vs = sp.shard_seq(Q, n), sp.shard_seq(K, n), sp.shard_seq(V, n)
        a = sp.ulysses_forward(Qs, Ks, Vs, attn)
        p = sp.pipesp_forward(Qs, Ks, Vs, H // n, attn)
        for x, y in zip(a, p):
            assert np.array_equal(x, y)


# ----------------------------------------------------------- Aco
@pytest.mark.parametrize("N_d,N_c,H", [(6, 2, 24), (1, 1, 2), (3, 1, 12), (2, 2, 8)])
def test_aco_relay_equals_unsharded(N_d, N_c, H):
    rng = np.random.default_rng(N_d * 10 + N_c)
    B, S, D = 1, 6 * N_d, 4
    Q, K, V = (rng.standard_normal((B, S, H, D)) for _ in range(3))
    ref = oracle.mha_unsharded(Q, K, V, nthreads=1)
    attn = lambda q, k, v: oracle.attention_rows(q, k, v, nthreads=1)  # noqa: E731
    outs = sp.aco_forward(sp.shard_seq(Q, N_d), sp.shard_seq(K, N_d), sp.shard_seq(V, N_d), N_c, attn)
    assert np.array_equal(np.concatenate(outs, axis=1), ref)


def test_aco_speedup_eq3_and_pad_heads(golden_dir):
    g = _golden(golden_dir)
    for key in ("aco_speedup", "aco_ideal_6_2"):
        assert abs(sp.aco_ideal_speedup(*g[key]["args"]) - g[key]["S"]) < 1e-12
    for H, n, Hp, pad in g["pad_heads"]:
        assert sp.pad_heads(H, n) == (Hp, pad)


def test_shard_bounds_differ_by_at_most_one():
    for S in (1, 7, 29, 118_800, 28_800):
        for P in (1, 2, 3, 6, 7, 8):
            if S < P:
                continue
            b = sp.shard_bounds(S, P)
            lens = np.diff(b)
            assert b[0] == 0 and b[-1] == S and lens.max() - lens.min() <= 1 and (np.diff(lens) <= 0).all()


@pytest.mark.parametrize("P,S,stages", [(3, 29, 1), (3, 29, 2), (7, 7 * 5 + 3, 1), (4, 4 * 6 + 3, 3), (2, 9, 2)])
def test_uneven_shards_pipesp_equals_unsharded(P, S, stages):
    """S % P != 0 (R9: shards differ by one token; the Aco example of PAPER.md:198 runs 7 denoising GPUs):
    Ulysses and PipeSP give unsharded attention bit for bit (same per-row routine, same data)."""
    rng = np.random.default_rng(P * 100 + S)
    B, H, D = 2, P * (3 if stages == 3 else 2), 4
    Q, K, V = (rng.standard_normal((B, S, H, D)) for _ in range(3))
    Qs, Ks, Vs = (sp.shard_seq(X, P, uneven=True) for X in (Q, K, V))
    ref = oracle.mha_unsharded(Q, K, V)
    assert np.array_equal(np.concatenate(sp.pipesp_forward(Qs, Ks, Vs, stages, oracle.attention_rows), axis=1), ref)
    assert np.array_equal(np.concatenate(sp.ulysses_forward(Qs, Ks, Vs, oracle.attention_rows), axis=1), ref)


def test_uneven_seq_to_head_labels():
    """Label routing: rank r's head block holds every source's tokens in sequence order (P=3, S=8)."""
    P, S, H = 3, 8, 3
    X = (np.arange(S)[None, :, None, None] * 10 + np.arange(H)[None, None, :, None]).astype(np.float64)
    R = sp.seq_to_head(sp.shard_seq(X, P, uneven=True))
    for r in range(P):
        assert np.array_equal(R[r][0, :, 0, 0], np.arange(S) * 10 + r)
    back = sp.head_to_seq(R)
    assert [x.shape[1] for x in back] == [3, 3, 2]
    assert np.array_equal(np.concatenate(back, axis=1), X)
