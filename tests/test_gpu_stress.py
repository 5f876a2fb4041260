"""Randomised and numerically hard GPU cases through the C ABI (seeded, reproducible).

* random plan shapes (P, H, D, B, S -- also not divisible by P --, stage count, head padding, key padding,
  staged or direct transport) -- PipeSP over P virtual ranks
  must give the same bits as the single-GPU kernel and stay within the north-star tolerance of the fp64
  oracle (R18/R19);
* large score ranges (Q scaled by powers of two, exact in bf16) that make the running max move often and by
  a lot (the conditional rescale, threshold 2^8) and drive most exponentials to underflow;
* Ring / USP on random shapes.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_12056_b200 import spa
from tests import gpu_util as U

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1200)]


def _shards(x, n):
    """sequence shards, uneven (first S % n ranks one token longer) when n does not divide S"""
    S, out, t = x.shape[1], [], 0
    for r in range(n):
        ln = S // n + (1 if r < S % n else 0)
        out.append(x[:, t:t + ln].contiguous())
        t += ln
    return out


def _oracle(q, k, v, kv_len=None):
    Q, K, V = (t.detach().cpu().double().numpy() for t in (q, k, v))
    kv = None if kv_len is None else oracle.key_valid_from_lengths(kv_len, K.shape[1])
    return oracle.mha_unsharded(Q, K, V, key_valid=kv)


def _case(seed):
    rng = np.random.default_rng(seed)
    P = int(rng.choice([1, 2, 3, 4, 6, 8]))
    D = int(rng.choice([64, 96, 128]))
    B = int(rng.integers(1, 3))
    S_l = int(rng.integers(1, 160))
    pad = bool(rng.integers(0, 2)) and P > 1
    h = int(rng.integers(1, 4))
    H = P * h - (int(rng.integers(1, P)) if pad and P > 1 else 0)
    H = max(H, 1)
    hp = -(-H // P)
    stages = int(rng.integers(1, 2 * hp + 1))
    while stages // np.gcd(stages, hp) > S_l:   # query chunks must not exceed local tokens
        stages -= 1
    masked = bool(rng.integers(0, 2))
    return P, H, D, B, S_l, max(stages, 1), pad, masked, rng


@pytest.mark.parametrize("seed", range(40))
def test_random_plans_bit_identical_and_within_tolerance(seed):
    P, H, D, B, S_l, stages, pad, masked, rng = _case(seed)
    S = S_l * P + int(rng.integers(0, P))      # uneven shards (R9) in about half the cases
    direct = bool(rng.integers(0, 2))          # SPA_OPT_DIRECT (f1 data path, loopback model)
    q, k, v = U.qkv(B, S, H, D, seed=1000 + seed)
    kv_len = None
    if masked:
        kv_len = torch.tensor([int(x) for x in rng.integers(0, S + 1, B)], dtype=torch.int32, device="cuda")
    single = spa.attention(q, k, v, kv_len=kv_len)
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages, pad_heads=pad)
    if kv_len is not None:
        plan.set_kv_len(kv_len)
    if direct:
        plan.set_option(spa.SPA_OPT_DIRECT, 1)
    qs, ks, vs = _shards(q, P), _shards(k, P), _shards(v, P)
    outs = [torch.full_like(t, float("nan")) for t in qs]
    spa.spa_pipesp_attention_local(plan, qs, ks, vs, outs, plan.workspace())
    torch.cuda.synchronize()
    out = torch.cat(outs, dim=1)
    assert torch.equal(out.view(torch.int16), single.view(torch.int16)), (P, H, D, B, S, stages, pad, masked, direct)
    U.assert_close(out, _oracle(q, k, v, None if kv_len is None else kv_len.tolist()))


@pytest.mark.parametrize("scale", [4.0, 16.0, 64.0])
@pytest.mark.parametrize("D", [96, 128])
def test_large_score_ranges(scale, D):
    """Scores spread over hundreds (log2 units): frequent large moves of the running max, most exps underflow
    to 0, a few keys dominate each row."""
    B, S, H = 1, 1500, 2
    q, k, v = U.qkv(B, S, H, D, seed=int(scale) + D)
    q = (q.float() * scale).to(torch.bfloat16)       # power-of-two scale: exact in bf16
    out = spa.attention(q, k, v)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    U.assert_close(out, _oracle(q, k, v))


def test_increasing_scores_force_rescale_every_tile():
    """K rows growing along the sequence: each new 128-key tile raises the row max by more than 2^8 (log2),
    so every tile takes the O-rescale path."""
    B, S, H, D = 1, 1280, 1, 128
    q, k, v = U.qkv(B, S, H, D, seed=7)
    q = torch.ones_like(q)
    ramp = torch.linspace(0, 1.0, S, device="cuda").view(1, S, 1, 1)
    k = (torch.ones_like(k).float() * ramp * 48.0).to(torch.bfloat16)   # score = sum_d k / sqrt(D): 0 .. ~543
    out = spa.attention(q, k, v)
    torch.cuda.synchronize()
    U.assert_close(out, _oracle(q, k, v))


@pytest.mark.parametrize("seed", range(4))
def test_random_ring_and_usp(seed):
    rng = np.random.default_rng(seed)
    P = int(rng.choice([2, 4, 6, 8]))
    Ud = int(rng.choice([d for d in (1, 2, 3, 4) if P % d == 0]))
    D = int(rng.choice([64, 96, 128]))
    H = Ud * int(rng.integers(1, 4))
    S_l = int(rng.integers(16, 150))
    B, S = 1, S_l * P
    q, k, v = U.qkv(B, S, H, D, seed=2000 + seed)
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, ring=True, ulysses=Ud)
    qs, ks, vs = _shards(q, P), _shards(k, P), _shards(v, P)
    outs = [torch.full_like(t, float("nan")) for t in qs]
    spa.spa_ring_attention_local(plan, qs, ks, vs, outs, plan.workspace())
    torch.cuda.synchronize()
    U.assert_close(torch.cat(outs, dim=1), _oracle(q, k, v))
