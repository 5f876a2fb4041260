"""Pins for the fp64 attention oracle (oracle/attention_oracle.c) against things that are
not the oracle: the SPEC worked example, closed forms, invariants, a library routine
(scipy softmax) and brute force in plain Python.  CPU only."""
import json
import math
import os

import numpy as np
import pytest
import scipy.special

import oracle


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def test_worked_example_spec69(golden_dir):
    g = _load(golden_dir, "attention_worked_example.json")
    out = oracle.attention_rows(np.array(g["Q"]), np.array(g["K"]), np.array(g["V"]))
    np.testing.assert_allclose(out, np.array(g["out"]), rtol=0, atol=4e-16)
    w = oracle.softmax_weights(np.array(g["Q"][0]), np.array(g["K"]))
    np.testing.assert_allclose(w, g["row0_weights"], rtol=0, atol=2e-16)


def test_scale_is_one_over_sqrt_d(golden_dir):
    g = _load(golden_dir, "scale_closed_form.json")
    out = oracle.attention_rows(np.array(g["q"]), np.array(g["K"]), np.array(g["V"]))
    np.testing.assert_allclose(out, g["out"], rtol=0, atol=4e-16)


def test_single_key_returns_v_exactly():
    rng = np.random.default_rng(1)
    for D in (1, 4, 64):
        q = rng.standard_normal((5, D))
        K = rng.standard_normal((1, D))
        V = rng.standard_normal((1, D))
        out = oracle.attention_rows(q, K, V)
        assert np.array_equal(out, np.repeat(V, 5, axis=0))  # softmax of a scalar is 1


@pytest.mark.parametrize("S,D", [(7, 3), (64, 16), (300, 96)])
def test_equal_keys_give_column_mean_of_v(S, D):
    """All K rows equal -> uniform weights -> column mean of V (north_star closed form)."""
    rng = np.random.default_rng(S + D)
    q = rng.standard_normal((4, D))
    K = np.repeat(rng.standard_normal((1, D)), S, axis=0)
    V = rng.standard_normal((S, D))
    out = oracle.attention_rows(q, K, V)
    mean = np.array([math.fsum(V[:, d]) / S for d in range(D)])
    np.testing.assert_allclose(out, np.broadcast_to(mean, out.shape), rtol=0, atol=1e-14)


def test_zero_query_gives_column_mean_of_v():
    rng = np.random.default_rng(3)
    S, D = 129, 8
    K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    out = oracle.attention_rows(np.zeros((2, D)), K, V)
    mean = np.array([math.fsum(V[:, d]) / S for d in range(D)])
    np.testing.assert_allclose(out, np.broadcast_to(mean, out.shape), rtol=0, atol=1e-14)


def test_rows_sum_to_one_and_convex():
    rng = np.random.default_rng(4)
    S, D = 257, 32
    K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    for sigma in (0.1, 1.0, 4.0, 30.0):
        q = sigma * rng.standard_normal(D)
        w = oracle.softmax_weights(q, K)
        assert abs(math.fsum(w) - 1.0) < 1e-12
        assert (w >= 0).all()
        out = oracle.attention_rows(q[None], K, V)[0]
        assert (out <= V.max(axis=0) + 1e-12).all() and (out >= V.min(axis=0) - 1e-12).all()


@pytest.mark.parametrize("S,D", [(5, 3), (33, 7), (128, 64)])
def test_matches_library_softmax(S, D):
    """Library routine (scipy.special.softmax + numpy matmul) on non-square, non-symmetric inputs:
    catches transposed operands, wrong scale, dropped max-subtraction."""
    rng = np.random.default_rng(S * 31 + D)
    Q, K, V = (rng.standard_normal((S + 3, D)), rng.standard_normal((S, D)), rng.standard_normal((S, D + 0)))
    ref = scipy.special.softmax(Q @ K.T / np.sqrt(D), axis=1) @ V
    out = oracle.attention_rows(Q, K, V)
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-13)


def test_brute_force_python():
    rng = np.random.default_rng(5)
    S, D = 9, 5
    Q, K, V = rng.standard_normal((S, D)), rng.standard_normal((S, D)), rng.standard_normal((S, D))
    out = oracle.attention_rows(Q, K, V)
    for s in range(S):
        z = [sum(Q[s, d] * K[t, d] for d in range(D)) / math.sqrt(D) for t in range(S)]
        m = max(z)
        e = [math.exp(x - m) for x in z]
        l = math.fsum(e)
        for d in range(D):
            ref = math.fsum(e[t] / l * V[t, d] for t in range(S))
            assert abs(out[s, d] - ref) < 1e-14


def test_shift_invariance_of_scores():
    """Adding one vector to every key shifts each row's scores by a constant -> same output."""
    rng = np.random.default_rng(6)
    S, D = 50, 16
    Q, K, V = rng.standard_normal((3, D)), rng.standard_normal((S, D)), rng.standard_normal((S, D))
    u = rng.standard_normal(D)
    np.testing.assert_allclose(oracle.attention_rows(Q, K + u, V), oracle.attention_rows(Q, K, V),
                               rtol=0, atol=1e-13)


def test_deterministic_and_thread_count_independent():
    rng = np.random.default_rng(7)
    S, D = 333, 24
    Q, K, V = rng.standard_normal((40, D)), rng.standard_normal((S, D)), rng.standard_normal((S, D))
    a = oracle.attention_rows(Q, K, V, nthreads=1)
    b = oracle.attention_rows(Q, K, V, nthreads=8)
    c = oracle.attention_rows(Q[17:18], K, V, nthreads=3)
    assert np.array_equal(a, b) and np.array_equal(a[17:18], c)


def test_mha_unsharded_is_per_head():
    rng = np.random.default_rng(8)
    B, S, H, D = 2, 16, 3, 4
    Q, K, V = (rng.standard_normal((B, S, H, D)) for _ in range(3))
    out = oracle.mha_unsharded(Q, K, V)
    for b in range(B):
        for k in range(H):
            ref = scipy.special.softmax(Q[b, :, k] @ K[b, :, k].T / 2.0, axis=1) @ V[b, :, k]
            np.testing.assert_allclose(out[b, :, k], ref, rtol=0, atol=1e-13)
