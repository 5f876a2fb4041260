"""Helpers for the -m gpu parity tests: inputs from synthgen, expected values from oracle/."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synthgen

MAX_ABS = 2e-2   # BASELINE.json north_star tolerance (bf16 inputs vs fp64 oracle)
REL_L2 = 5e-3


def qkv(B, S, H, D, seed=0, dist="D0", device="cuda"):
    shape = (B, S, H, D)
    return [synthgen.gen_qkv_shard(seed, t, shape, 0, S, dist=dist).to(device)
            for t in (synthgen.TENSOR_Q, synthgen.TENSOR_K, synthgen.TENSOR_V)]


def oracle_mha(q, k, v, nthreads=None) -> np.ndarray:
    """fp64 oracle on the exact bf16 values (bf16 -> fp64 is exact)."""
    Q, K, V = (t.detach().cpu().double().numpy() for t in (q, k, v))
    return oracle.mha_unsharded(Q, K, V, nthreads)


def oracle_rows(q, k, v, b, head, rows) -> np.ndarray:
    Q = q[b, rows, head].detach().cpu().double().numpy()
    K = k[b, :, head].detach().cpu().double().numpy()
    V = v[b, :, head].detach().cpu().double().numpy()
    return oracle.attention_rows(Q, K, V)


def errors(out: torch.Tensor, ref: np.ndarray):
    o = out.detach().cpu().double().numpy()
    diff = o - ref
    max_abs = float(np.abs(diff).max())
    rel = float(np.linalg.norm(diff.ravel()) / max(np.linalg.norm(ref.ravel()), 1e-300))
    return max_abs, rel


def assert_close(out, ref, max_abs=MAX_ABS, rel_l2=REL_L2):
    ma, rl = errors(out, ref)
    assert ma <= max_abs and rl <= rel_l2, f"max_abs={ma:.3e} rel_l2={rl:.3e}"
    return ma, rl
