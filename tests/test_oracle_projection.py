"""Pins of oracle/projection.py (the QKV projections) against things other than itself:
plain-Python brute force, one-hot closed forms, a labelled weight that identifies every (tensor, head, dim)
slot of the fused layout, linearity, torch's own fp32 -> bf16 rounding, and hand-worked rounding cases."""
import math

import numpy as np
import pytest
import torch

from oracle import projection as pj
from oracle import sp
import oracle


def _bf16_vals(rng, shape, scale=1.0):
    """Random values that are exactly bf16 (so fp64 holds them exactly), like the GPU inputs."""
    x = torch.from_numpy(rng.standard_normal(shape) * scale).to(torch.bfloat16)
    return x.double().numpy()


# ---------------------------------------------------------------- bf16 rounding
@pytest.mark.parametrize("x,expect", [
    (1.0, 1.0),
    (1.0 + 2 ** -8, 1.0),                      # halfway 1 | 1+2^-7: ties to even -> 1
    (1.0 + 3 * 2 ** -8, 1.0 + 2 ** -6),        # halfway 1+2^-7 | 1+2^-6: even mantissa is 1+2^-6
    (1.0 + 2 ** -8 + 2 ** -40, 1.0 + 2 ** -7),  # just above halfway (a double-rounding trap via fp32)
    (-3.0 - 2 ** -7, -3.0),                    # spacing 2^-6 in [2,4): -3-2^-7 is halfway -> even (-3)
    (255.5, 256.0),                            # 255.5 lies between 255 and 256 (spacing 1): halfway -> even 256
    (2.0 ** -130, 2.0 ** -130),                # bf16 subnormal, exactly representable
    (0.0, 0.0),
])
def test_bf16_round_hand_cases(x, expect):
    assert pj.bf16_round(np.array([x]))[0] == expect


def test_bf16_round_matches_torch_on_fp32_values():
    """On values exactly representable in fp32 the fp64 -> bf16 rounding equals torch's fp32 -> bf16 (RNE)."""
    rng = np.random.default_rng(0)
    x32 = (rng.standard_normal(200_000) * np.exp(rng.uniform(-20, 20, 200_000))).astype(np.float32)
    ours = pj.bf16_round(x32.astype(np.float64))
    theirs = torch.from_numpy(x32).to(torch.bfloat16).double().numpy()
    assert np.array_equal(ours, theirs)


def test_bf16_round_nearest_property():
    """|x - bf16(x)| <= half an ulp of the bf16 grid at x, and the result has at most 8 significant bits."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal(50_000) * 10.0 ** rng.uniform(-5, 5, 50_000)
    y = pj.bf16_round(x)
    ulp = np.ldexp(1.0, np.frexp(np.abs(x))[1] - 8)
    assert np.all(np.abs(x - y) <= ulp / 2)
    m, _ = np.frexp(y)
    assert np.all(np.rint(m * 256) == m * 256)


# ---------------------------------------------------------------- the projection
def test_brute_force_tiny():
    """Plain-Python loops with math.fsum (exactly rounded sums) on a tiny problem, fp64 (no bf16 rounding)."""
    rng = np.random.default_rng(2)
    B, S, C, H, D = 2, 3, 5, 2, 4
    X = _bf16_vals(rng, (B, S, C))
    W = _bf16_vals(rng, (3 * H * D, C))
    bias = rng.standard_normal(3 * H * D)
    Q, K, V = pj.qkv_projection(X, W, bias, H, D, round_bf16=False)
    outs = (Q, K, V)
    for b in range(B):
        for s in range(S):
            for t in range(3):
                for k in range(H):
                    for d in range(D):
                        o = t * H * D + k * D + d
                        ref = math.fsum([X[b, s, c] * W[o, c] for c in range(C)] + [bias[o]])
                        assert abs(outs[t][b, s, k, d] - ref) <= 1e-14 * (1 + abs(ref))


def test_one_hot_inputs_select_weight_columns():
    """X = e_c (one-hot over the hidden dim) -> every output is exactly W[o, c] (+ bias): a closed form."""
    rng = np.random.default_rng(3)
    C, H, D = 8, 3, 4
    W = _bf16_vals(rng, (3 * H * D, C))
    bias = _bf16_vals(rng, (3 * H * D,))
    X = np.eye(C)[None]                       # [1, C tokens, C]: token s is e_s
    Q, K, V = pj.qkv_projection(X, W, bias, H, D)
    for s in range(C):
        for t, T in enumerate((Q, K, V)):
            exact = W[t * H * D:(t + 1) * H * D, s] + bias[t * H * D:(t + 1) * H * D]
            assert np.array_equal(exact.astype(np.float32).astype(np.float64), exact)   # fp32 holds the sum
            ref = torch.from_numpy(exact.astype(np.float32)).to(torch.bfloat16).double().numpy()   # torch's RNE
            assert np.array_equal(T[0, s].reshape(-1), ref)
    Q0, _, _ = pj.qkv_projection(X, W, None, H, D)    # without bias: exactly the (bf16) weight column
    assert np.array_equal(Q0[0, 2].reshape(-1), W[:H * D, 2])


def test_labelled_weight_routes_every_slot():
    """W[o] = (o + 1) * e_0 and X = e_0: output (t, k, d) must read o + 1 = t*H*D + k*D + d + 1 -- catches any
    transposed tensor / head / dim index in the fused layout."""
    H, D, C = 3, 8, 4
    W = np.zeros((3 * H * D, C))
    W[:, 0] = np.arange(1, 3 * H * D + 1)
    X = np.zeros((1, 1, C))
    X[0, 0, 0] = 1.0
    Q, K, V = pj.qkv_projection(X, W, None, H, D)
    for t, T in enumerate((Q, K, V)):
        for k in range(H):
            for d in range(D):
                assert T[0, 0, k, d] == t * H * D + k * D + d + 1


def test_bias_only_and_linearity():
    rng = np.random.default_rng(4)
    B, S, C, H, D = 1, 6, 16, 2, 8
    W = _bf16_vals(rng, (3 * H * D, C))
    bias = rng.standard_normal(3 * H * D)
    Q, K, V = pj.qkv_projection(np.zeros((B, S, C)), W, bias, H, D, round_bf16=False)
    assert np.array_equal(Q[0, 3].reshape(-1), bias[:H * D]) and np.array_equal(V[0, 5].reshape(-1), bias[2 * H * D:])
    X1, X2 = _bf16_vals(rng, (B, S, C)), _bf16_vals(rng, (B, S, C))
    a = pj.qkv_projection(2.0 * X1 - 0.5 * X2, W, None, H, D, round_bf16=False)
    b1 = pj.qkv_projection(X1, W, None, H, D, round_bf16=False)
    b2 = pj.qkv_projection(X2, W, None, H, D, round_bf16=False)
    for t in range(3):
        assert np.allclose(a[t], 2.0 * b1[t] - 0.5 * b2[t], rtol=0, atol=1e-12)


def test_pipesp_qkv_equals_unsharded():
    """Projecting each sequence shard and running PipeSP = projecting the whole sequence and running
    unsharded attention, bit for bit in fp64 (rows are independent)."""
    rng = np.random.default_rng(5)
    B, S, C, H, D, P = 1, 32, 24, 4, 8, 2
    X = _bf16_vals(rng, (B, S, C), 0.5)
    W = _bf16_vals(rng, (3 * H * D, C), 0.3)
    bias = rng.standard_normal(3 * H * D) * 0.1
    attn = lambda q, k, v: oracle.attention_rows(q, k, v, 1)   # noqa: E731
    Xs = [X[:, r * S // P:(r + 1) * S // P] for r in range(P)]
    for n_st in (1, 2):
        outs = pj.pipesp_qkv_forward(Xs, W, bias, H, D, n_st, attn)
        Q, K, V = pj.qkv_projection(X, W, bias, H, D)
        ref = oracle.mha_unsharded(Q, K, V, 1)
        assert np.array_equal(np.concatenate(outs, axis=1), ref)
