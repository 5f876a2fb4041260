"""Seeded synthetic Q/K/V generator shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no attention, no reshard,
no all-to-all).  It only turns (seed, tensor id, global element index) into a
bf16 bit pattern, so that the CPU oracle and the GPU path see identical inputs
and every rank can generate just its own shard.

Recipe (SURVEY.md §8(d) "Value distributions"):

    u_i  = (splitmix64(key(seed, tensor_id, 4*flat + i)) >> 40) * 2^-24,  i = 0..3
    IH4  = (u_0 + u_1 + u_2 + u_3 - 2) * sqrt(3)           # Irwin-Hall ~ N(0,1)
    x    = bf16_rne(f32_rne(sigma * IH4))

``flat`` is the row-major index of the element in the GLOBAL unsharded
[B, S, H, D] tensor, so a shard / a single head / a single token row is
generated bit-identically to the same elements of the full tensor.

Everything is integer arithmetic plus IEEE fp64 mul/add evaluated one torch op
at a time, so CPU and CUDA produce the same bits.

Distributions:
  D0  i.i.d. sigma=1 for Q, K, V                      (perf workload)
  D1  "peaky": sigma_Q = 4, K, V sigma = 1
  D2  Q == 0 (closed form: output = column mean of V)
  D3  V == 1 (normalisation: output == 1)
  D4  "video-locality": K = bf16(Q + 0.5 * noise)
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import torch

__all__ = [
    "TENSOR_Q", "TENSOR_K", "TENSOR_V",
    "splitmix64", "uniform24", "irwin_hall4", "bf16_bits_from_f64",
    "gen_elements", "gen_qkv_shard", "gen_head_rows", "bf16_bits_to_f64",
    "Workload", "WORKLOADS", "tokens_for_video",
    "TENSOR_X", "TENSOR_W", "TENSOR_BIAS", "gen_hidden_shard", "gen_qkv_weight", "gen_qkv_bias",
]

TENSOR_Q, TENSOR_K, TENSOR_V = 0, 1, 2
_NOISE_K = 3  # D4 noise stream
TENSOR_X, TENSOR_W, TENSOR_BIAS = 4, 5, 6   # hidden states, fused QKV weight, its bias (QKV projection, f3)

_M64 = (1 << 64)


def _s64(c: int) -> int:
    """Unsigned 64-bit constant -> the int64 with the same bits."""
    c &= _M64 - 1
    return c - _M64 if c >= (1 << 63) else c


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_MIX1 = _s64(0xBF58476D1CE4E5B9)
_MIX2 = _s64(0x94D049BB133111EB)


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical shift right of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrapping two's-complement arithmetic)."""
    z = x + _GOLDEN
    z = (z ^ _lsr(z, 30)) * _MIX1
    z = (z ^ _lsr(z, 27)) * _MIX2
    return z ^ _lsr(z, 31)


def _key(seed: int, tensor_id: int, counter: torch.Tensor) -> torch.Tensor:
    assert 0 <= seed < (1 << 11) and 0 <= tensor_id < (1 << 8)
    return counter + ((seed << 52) | (tensor_id << 44))


def uniform24(seed: int, tensor_id: int, counter: torch.Tensor) -> torch.Tensor:
    """u in [0,1) with 24 random bits, as float64 (exact)."""
    bits = _lsr(splitmix64(_key(seed, tensor_id, counter)), 40)
    return bits.to(torch.float64) * (2.0 ** -24)


def irwin_hall4(seed: int, tensor_id: int, flat: torch.Tensor) -> torch.Tensor:
    """(u0+u1+u2+u3-2)*sqrt(3): mean 0, variance 1 (fp64, op by op)."""
    base = flat * 4
    s = uniform24(seed, tensor_id, base)
    for i in range(1, 4):
        s = s + uniform24(seed, tensor_id, base + i)
    return (s - 2.0) * math.sqrt(3.0)


def bf16_bits_from_f64(x: torch.Tensor) -> torch.Tensor:
    """fp64 -> fp32 (IEEE RNE) -> bf16 (RNE on the fp32 bit pattern); returns int16 bits.

    Inputs are finite and far from overflow, so no NaN/Inf handling is needed.
    """
    b = x.to(torch.float32).view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    rounded = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    rounded = rounded & 0xFFFF
    return torch.where(rounded >= 0x8000, rounded - 0x10000, rounded).to(torch.int16)


def bf16_bits_to_f64(bits: torch.Tensor) -> torch.Tensor:
    """Exact bf16 bit pattern (int16/uint16/bfloat16 tensor) -> float64."""
    if bits.dtype == torch.bfloat16:
        bits = bits.view(torch.int16)
    b32 = (bits.to(torch.int32) & 0xFFFF) << 16
    return b32.view(torch.float32).to(torch.float64)


def _flat_index(shape_global: Tuple[int, int, int, int], b: torch.Tensor, s: torch.Tensor,
                k: torch.Tensor, d: torch.Tensor) -> torch.Tensor:
    B, S, H, D = shape_global
    return ((b * S + s) * H + k) * D + d


def gen_elements(seed: int, tensor_id: int, dist: str, flat: torch.Tensor,
                 q_flat_noise: bool = False) -> torch.Tensor:
    """bf16 bits (int16) for the given global flat indices of tensor `tensor_id` under `dist`."""
    dist = dist.upper()
    if dist not in ("D0", "D1", "D2", "D3", "D4"):
        raise ValueError(f"unknown distribution {dist}")
    if dist == "D2" and tensor_id == TENSOR_Q:
        return torch.zeros_like(flat, dtype=torch.int16)
    if dist == "D3" and tensor_id == TENSOR_V:
        return torch.full_like(flat, 0x3F80, dtype=torch.int16)  # bf16(1.0)
    if dist == "D4" and tensor_id == TENSOR_K:
        q = bf16_bits_to_f64(gen_elements(seed, TENSOR_Q, "D0", flat))
        noise = irwin_hall4(seed, _NOISE_K, flat)
        return bf16_bits_from_f64(q + 0.5 * noise)
    sigma = 4.0 if (dist == "D1" and tensor_id == TENSOR_Q) else 1.0
    return bf16_bits_from_f64(sigma * irwin_hall4(seed, tensor_id, flat))


def gen_qkv_shard(seed: int, tensor_id: int, shape_global: Sequence[int], tok0: int, tok1: int,
                  dist: str = "D0", device="cpu", chunk_elems: int = 1 << 26) -> torch.Tensor:
    """Rows [tok0, tok1) of the global [B,S,H,D] tensor as a contiguous bf16 [B, tok1-tok0, H, D]."""
    B, S, H, D = shape_global
    n_tok = tok1 - tok0
    out = torch.empty((B, n_tok, H, D), dtype=torch.int16, device=device)
    flat_out = out.view(-1)
    per_tok = H * D
    rows_per_chunk = max(1, chunk_elems // per_tok)
    for b in range(B):
        for t0 in range(0, n_tok, rows_per_chunk):
            t1 = min(n_tok, t0 + rows_per_chunk)
            start = ((b * S) + tok0 + t0) * per_tok
            flat = torch.arange(start, start + (t1 - t0) * per_tok, device=device, dtype=torch.int64)
            o0 = (b * n_tok + t0) * per_tok
            flat_out[o0:o0 + flat.numel()] = gen_elements(seed, tensor_id, dist, flat)
    return out.view(torch.bfloat16)


def gen_head_rows(seed: int, tensor_id: int, shape_global: Sequence[int], b: int, head: int,
                  tokens: Optional[torch.Tensor] = None, dist: str = "D0", device="cpu") -> torch.Tensor:
    """bf16 [T, D] of one (batch, head): all S tokens, or the given token indices."""
    B, S, H, D = shape_global
    if tokens is None:
        tokens = torch.arange(S, device=device, dtype=torch.int64)
    tokens = tokens.to(device=device, dtype=torch.int64)
    d = torch.arange(D, device=device, dtype=torch.int64)
    flat = _flat_index((B, S, H, D), torch.tensor(b, device=device), tokens[:, None],
                       torch.tensor(head, device=device), d[None, :])
    return gen_elements(seed, tensor_id, dist, flat).view(torch.bfloat16)


def tokens_for_video(width: int, height: int, frames: int) -> int:
    """Latent tokens for a 4x8x8 VAE and 1x2x2 patch (an assumption, not the paper's)."""
    return ((frames - 1) // 4 + 1) * (height // 16) * (width // 16)


@dataclass(frozen=True)
class Workload:
    name: str
    B: int
    S: int
    H: int
    D: int


# BASELINE.json "configs" (shapes only; P is a run parameter)
WORKLOADS = {
    "tiny": Workload("tiny", 1, 256, 4, 64),
    "osp480p93f": Workload("osp480p93f", 1, 28_800, 24, 96),
    "hy544p129f": Workload("hy544p129f", 1, 76_032, 24, 128),
    "hy720p129f": Workload("hy720p129f", 1, 118_800, 24, 128),
}


# ------------------------------------------------------------------ hidden states / QKV weights
def _gen_flat(seed: int, tensor_id: int, n: int, sigma: float, device, start: int = 0,
              chunk: int = 1 << 26) -> torch.Tensor:
    """bf16 bits of sigma*IH4 for flat indices [start, start+n) of tensor `tensor_id` (int16 [n])."""
    out = torch.empty(n, dtype=torch.int16, device=device)
    for i in range(0, n, chunk):
        j = min(n, i + chunk)
        flat = torch.arange(start + i, start + j, device=device, dtype=torch.int64)
        out[i:j] = bf16_bits_from_f64(sigma * irwin_hall4(seed, tensor_id, flat))
    return out


def gen_hidden_shard(seed: int, shape_global: Sequence[int], tok0: int, tok1: int, device="cpu") -> torch.Tensor:
    """Rows [tok0, tok1) of the global hidden states X [B, S, C] (sigma = 1: LayerNorm-ed DiT activations)."""
    B, S, C = shape_global
    n = tok1 - tok0
    out = torch.empty((B, n, C), dtype=torch.int16, device=device)
    for b in range(B):
        out[b].view(-1).copy_(_gen_flat(seed, TENSOR_X, n * C, 1.0, device, start=(b * S + tok0) * C))
    return out.view(torch.bfloat16)


def gen_qkv_weight(seed: int, C: int, H: int, D: int, device="cpu") -> torch.Tensor:
    """Fused nn.Linear weight W [3*H*D, C] bf16, sigma = 1/sqrt(C) (variance-preserving init: Q, K, V ~ N(0, 1))."""
    return _gen_flat(seed, TENSOR_W, 3 * H * D * C, 1.0 / math.sqrt(C), device).view(3 * H * D, C).view(torch.bfloat16)


def gen_qkv_bias(seed: int, H: int, D: int, device="cpu") -> torch.Tensor:
    """Bias [3*H*D] as fp32 values of bf16 numbers, sigma = 0.1."""
    return _gen_flat(seed, TENSOR_BIAS, 3 * H * D, 0.1, device).view(torch.bfloat16).float()
