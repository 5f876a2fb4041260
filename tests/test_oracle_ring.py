"""Pins for the ring-attention pieces of the oracle (R21; PAPER.md:171 names Ring-Attention as the
fallback when H is not divisible by the GPU count but gives no procedure): the per-row log-sum-exp against
scipy.special.logsumexp, the lse merge against attention over the union of the key blocks (the softmax of a
concatenation), and the full ring over P virtual ranks against unsharded attention.  CPU only."""
import math

import numpy as np
import pytest
import scipy.special

import oracle
from oracle import sp


def test_lse_matches_scipy_logsumexp():
    rng = np.random.default_rng(3)
    S, D = 57, 16
    q = rng.standard_normal((5, D)) * 3
    K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    out, lse = oracle.attention_rows_lse(q, K, V)
    ref = scipy.special.logsumexp(q @ K.T / math.sqrt(D), axis=1)
    np.testing.assert_allclose(lse, ref, rtol=0, atol=1e-12)
    assert np.array_equal(out, oracle.attention_rows(q, K, V))


def test_lse_single_key_and_masked():
    rng = np.random.default_rng(4)
    D = 4
    q, k, v = rng.standard_normal((1, D)), rng.standard_normal((1, D)), rng.standard_normal((1, D))
    _, lse = oracle.attention_rows_lse(q, k, v)
    np.testing.assert_allclose(lse[0], float(q[0] @ k[0]) / 2.0, rtol=0, atol=1e-15)   # ln e^z = z, sqrt(4) = 2
    out, lse = oracle.attention_rows_lse(q, k, v, key_valid=np.zeros(1, bool))
    assert lse[0] == -np.inf and np.array_equal(out, np.zeros((1, D)))


@pytest.mark.parametrize("nblocks", [1, 2, 3, 7])
def test_lse_merge_of_disjoint_blocks_is_softmax_of_union(nblocks):
    rng = np.random.default_rng(nblocks)
    S, D = 7 * 6, 8
    q = rng.standard_normal((4, D)) * 2
    K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    cuts = np.linspace(0, S, nblocks + 1).astype(int)
    parts, lses = [], []
    for a, b in zip(cuts[:-1], cuts[1:]):
        o, l = oracle.attention_rows_lse(q, K[a:b], V[a:b])
        parts.append(o)
        lses.append(l)
    out, lse = sp.lse_merge(parts, lses)
    full, full_lse = oracle.attention_rows_lse(q, K, V)
    np.testing.assert_allclose(out, full, rtol=0, atol=1e-13)
    np.testing.assert_allclose(lse, full_lse, rtol=0, atol=1e-12)
    if nblocks == 1:
        assert np.array_equal(out, full)   # a single block merges to itself exactly (weight exp(0) = 1)


def test_lse_merge_with_empty_blocks():
    parts = [np.ones((2, 3)), np.full((2, 3), 5.0)]
    lses = [np.array([0.0, -np.inf]), np.array([-np.inf, -np.inf])]
    out, lse = sp.lse_merge(parts, lses)
    assert np.array_equal(out[0], np.ones(3)) and np.array_equal(out[1], np.zeros(3))
    assert lse[0] == 0.0 and lse[1] == -np.inf


@pytest.mark.parametrize("P,H", [(1, 3), (2, 3), (3, 2), (4, 5)])
def test_ring_equals_unsharded_any_head_count(P, H):
    """Ring attention needs no H % P == 0 (the reason the paper switches to it)."""
    rng = np.random.default_rng(P * 10 + H)
    B, S_l, D = 2, 5, 4
    S = S_l * P
    Q, K, V = (rng.standard_normal((B, S, H, D)) for _ in range(3))
    outs = sp.ring_forward(sp.shard_seq(Q, P), sp.shard_seq(K, P), sp.shard_seq(V, P), oracle.attention_rows_lse)
    np.testing.assert_allclose(np.concatenate(outs, axis=1), oracle.mha_unsharded(Q, K, V), rtol=0, atol=1e-13)


@pytest.mark.parametrize("P,U,H", [(4, 2, 2), (4, 2, 6), (6, 3, 3), (8, 4, 4), (4, 4, 4), (4, 1, 3)])
def test_usp_hybrid_equals_unsharded(P, U, H):
    """Ulysses degree U x Ring degree P/U = unsharded attention; U = P is plain Ulysses with a
    single-block ring, U = 1 plain Ring."""
    rng = np.random.default_rng(P * 100 + U * 10 + H)
    B, S_l, D = 1, 3, 4
    S = S_l * P
    Q, K, V = (rng.standard_normal((B, S, H, D)) for _ in range(3))
    outs = sp.usp_forward(sp.shard_seq(Q, P), sp.shard_seq(K, P), sp.shard_seq(V, P), U, oracle.attention_rows_lse)
    np.testing.assert_allclose(np.concatenate(outs, axis=1), oracle.mha_unsharded(Q, K, V), rtol=0, atol=1e-13)
