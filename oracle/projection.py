"""QKV linear projections of a DiT block (TEST INFRASTRUCTURE ONLY).

Definition followed (§3.3 "Linear projections: Q = X W_Q, K = X W_K, V = X W_V";
the projection whose computation OpenSoraPlan's PipeSP overlaps with the three input All-to-Alls,
PAPER.md:439 (§4.5)).  Weights use the fused nn.Linear layout of a DiT attention block:

    W      [3*H*D, C]    output feature o = t*H*D + k*D + d   (t = 0 Q, 1 K, 2 V; head k; dim d)
    bias   [3*H*D]       (optional)
    Y[b, s, o] = sum_c X[b, s, c] * W[o, c] + bias[o]      (fp64; numpy matmul as the library primitive)
    Q[b, s, k, d] = Y[b, s, 0*H*D + k*D + d], K = ... 1*H*D ..., V = ... 2*H*D ...

Precision reading (R22; the paper states none): X, W bf16 (exact in fp64), bias fp32; the
projections are stored as bf16 activations, i.e. the fp64 result rounded ONCE to bf16 (round to nearest,
ties to even) -- ``bf16_round`` below, then the attention oracle runs on those bf16 values.

Pinned by tests/test_oracle_projection.py against plain-Python brute force, one-hot closed forms, a
labelled weight that identifies every (t, k, d) slot, linearity, and torch's own fp32 -> bf16 rounding.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import numpy as np

from . import sp


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp64 -> nearest bf16 value (8 significant bits, ties to even), returned as fp64.

    One rounding step directly from fp64 (no intermediate fp32): x = m * 2^e with 0.5 <= |m| < 1, the
    significand m * 2^8 is rounded half-to-even (np.rint) and scaled back.  Values below the smallest
    normal bf16 (2^-126) round on the subnormal grid 2^-133.  Finite inputs only (no overflow handling:
    activations here are O(1e2) at most)."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    e = np.maximum(e, -125)                     # 2^-126 = 0.5 * 2^-125: below it the grid spacing stays 2^-133
    scale = np.ldexp(1.0, 8 - e)                # exact powers of two
    return np.rint(x * scale) / scale


def qkv_projection(X: np.ndarray, W: np.ndarray, bias: Optional[np.ndarray], H: int, D: int,
                   round_bf16: bool = True) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """X [B, S, C] (fp64 of bf16 values), W [3HD, C], bias [3HD] or None -> Q, K, V [B, S, H, D] (fp64).

    Y = X W^T + bias in fp64, split into the three tensors and heads by the fused layout
    above; rounded to bf16 unless round_bf16=False."""
    X = np.asarray(X, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    B, S, C = X.shape
    assert W.shape == (3 * H * D, C), W.shape
    Y = X.reshape(B * S, C) @ W.T
    if bias is not None:
        Y = Y + np.asarray(bias, dtype=np.float64)[None, :]
    if round_bf16:
        Y = bf16_round(Y)
    Y = Y.reshape(B, S, 3, H, D)
    return Y[:, :, 0].copy(), Y[:, :, 1].copy(), Y[:, :, 2].copy()


def pipesp_qkv_forward(Xs: List[np.ndarray], W: np.ndarray, bias: Optional[np.ndarray], H: int, D: int,
                       n_stages: int, attn) -> List[np.ndarray]:
    """The SP layer from the hidden states ("after each GPU computes its portion of the
    sub-sequence's Q, K and V, three rounds of All-to-All ..."): every rank projects its own sequence shard
    X_r [B, S_r, C] (bf16-rounded, as stored), then PipeSP (oracle.sp.pipesp_forward) on the projected shards.
    Overlapping the projection with the all-to-alls changes no value."""
    shards = [qkv_projection(X, W, bias, H, D) for X in Xs]
    Qs, Ks, Vs = ([s[i] for s in shards] for i in range(3))
    return sp.pipesp_forward(Qs, Ks, Vs, n_stages, attn)
