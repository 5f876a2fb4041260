"""Pins for the key-padding mask of the fp64 oracle (Alg. 1 `attention_mask`, PAPER.md:85/90;
DESIGN.md R20) and for the head-padding path, against things that are not
the oracle: brute force in plain Python on the truncated key set, scipy softmax on the selected keys,
the closed form Q = 0 -> mean of the valid V rows, and invariants.  CPU only."""
import math

import numpy as np
import pytest
import scipy.special

import oracle
from oracle import sp


def _brute(q, K, V):
    """plain-Python softmax attention of one row (no numpy reductions)."""
    D = len(q)
    z = [sum(q[d] * K[t][d] for d in range(D)) / math.sqrt(D) for t in range(len(K))]
    m = max(z)
    e = [math.exp(x - m) for x in z]
    l = math.fsum(e)
    return [math.fsum(e[t] / l * V[t][d] for t in range(len(K))) for d in range(D)]


@pytest.mark.parametrize("S,L", [(9, 1), (9, 5), (40, 39), (40, 40)])
def test_prefix_mask_equals_truncated_keys_brute_force(S, L):
    rng = np.random.default_rng(S * 100 + L)
    D = 6
    q = rng.standard_normal((3, D))
    K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    valid = oracle.key_valid_from_lengths([L], S)[0]
    out = oracle.attention_rows(q, K, V, key_valid=valid)
    for r in range(3):
        ref = _brute(list(q[r]), K[:L].tolist(), V[:L].tolist())
        np.testing.assert_allclose(out[r], ref, rtol=0, atol=1e-14)


def test_general_mask_matches_scipy_softmax_on_selected_keys():
    rng = np.random.default_rng(7)
    S, D = 50, 8
    q = rng.standard_normal((4, D))
    K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    valid = rng.random(S) < 0.4
    valid[3] = True
    out = oracle.attention_rows(q, K, V, key_valid=valid)
    w = scipy.special.softmax(q @ K[valid].T / math.sqrt(D), axis=1)
    np.testing.assert_allclose(out, w @ V[valid], rtol=0, atol=1e-13)


def test_zero_query_gives_mean_of_valid_values():
    rng = np.random.default_rng(11)
    S, D, L = 33, 5, 17
    K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    out = oracle.attention_rows(np.zeros((2, D)), K, V, key_valid=oracle.key_valid_from_lengths([L], S)[0])
    mean = [math.fsum(V[:L, d]) / L for d in range(D)]
    np.testing.assert_allclose(out, np.broadcast_to(mean, out.shape), rtol=0, atol=1e-15)


def test_masked_key_values_do_not_matter():
    """What sits at a masked position (huge scores, huge values) has no effect on the result."""
    rng = np.random.default_rng(5)
    S, D, L = 20, 4, 12
    q = rng.standard_normal((3, D))
    K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    valid = oracle.key_valid_from_lengths([L], S)[0]
    a = oracle.attention_rows(q, K, V, key_valid=valid)
    K2, V2 = K.copy(), V.copy()
    K2[L:] = 1e4
    V2[L:] = -1e6
    b = oracle.attention_rows(q, K2, V2, key_valid=valid)
    assert np.array_equal(a, b)


def test_no_valid_key_gives_zero_row_and_all_valid_is_unmasked():
    rng = np.random.default_rng(2)
    S, D = 10, 4
    q = rng.standard_normal((2, D))
    K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    assert np.array_equal(oracle.attention_rows(q, K, V, key_valid=np.zeros(S, bool)), np.zeros((2, D)))
    assert np.array_equal(oracle.attention_rows(q, K, V, key_valid=np.ones(S, bool)), oracle.attention_rows(q, K, V))


def test_mha_mask_is_per_batch_entry():
    rng = np.random.default_rng(9)
    B, S, H, D = 2, 12, 2, 4
    Q, K, V = (rng.standard_normal((B, S, H, D)) for _ in range(3))
    kv_len = [5, 12]
    out = oracle.mha_unsharded(Q, K, V, key_valid=oracle.key_valid_from_lengths(kv_len, S))
    for b in range(B):
        ref = oracle.mha_unsharded(Q[b:b + 1, :, :, :], K[b:b + 1, :kv_len[b]], V[b:b + 1, :kv_len[b]])
        # truncating K/V is the definition of a prefix mask; the query rows are all kept
        np.testing.assert_allclose(out[b], ref[0], rtol=0, atol=1e-14)


@pytest.mark.parametrize("H,P,stages", [(6, 4, 1), (6, 4, 2), (5, 2, 3), (24, 7, 1)])
def test_head_padding_equals_unsharded(H, P, stages):
    """H=24 over 7 ranks pads to 28 heads; the real heads' result is unsharded attention."""
    rng = np.random.default_rng(H * 10 + P)
    B, S_l, D = 1, 3, 4
    S = S_l * P
    Q, K, V = (rng.standard_normal((B, S, H, D)) for _ in range(3))
    Qs, Ks, Vs = (sp.shard_seq(X, P) for X in (Q, K, V))
    Hp, n_pad = sp.pad_heads(H, P)
    assert Hp % P == 0 and 0 < n_pad < P
    fwd = (lambda a, b, c: sp.pipesp_forward(a, b, c, stages, oracle.attention_rows))
    outs = sp.padded_forward(Qs, Ks, Vs, P, fwd)
    assert all(o.shape == (B, S_l, H, D) for o in outs)
    assert np.array_equal(np.concatenate(outs, axis=1), oracle.mha_unsharded(Q, K, V))


def test_zero_pad_head_gives_zero_output():
    """A pad head has Q = K = V = 0: uniform weights over zero values -> exactly 0 (closed form)."""
    S, D = 7, 4
    out = oracle.attention_rows(np.zeros((S, D)), np.zeros((S, D)), np.zeros((S, D)))
    assert np.array_equal(out, np.zeros((S, D)))
