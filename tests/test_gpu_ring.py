"""Ring attention (shape.ring = 1; PAPER.md:171 Ring-Attention fallback, R21) over P virtual ranks on one
GPU through the C ABI: the tcgen05 kernel's fp32 partials + per-row log-sum-exp merged by the lse-merge kernel,
vs the fp64 oracle (unsharded attention; oracle.sp.ring_forward is pinned equal to it), for head counts that
Ulysses cannot split."""
import pytest
import torch

import oracle

from paper_2511_12056_b200 import spa
from tests import gpu_util as U

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


def _shards(x, n):
    S_l = x.shape[1] // n
    return [x[:, r * S_l:(r + 1) * S_l].contiguous() for r in range(n)]


def _ring(P, q, k, v):
    B, S, H, D = q.shape
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, ring=True)
    qs, ks, vs = _shards(q, P), _shards(k, P), _shards(v, P)
    outs = [torch.full_like(t, float("nan")) for t in qs]
    ws = plan.workspace()
    spa.spa_ring_attention_local(plan, qs, ks, vs, outs, ws)
    torch.cuda.synchronize()
    return torch.cat(outs, dim=1)


@pytest.mark.parametrize("P,H,D", [(1, 3, 64), (2, 3, 128), (3, 2, 96), (4, 5, 96), (8, 24, 128), (7, 24, 64)])
def test_ring_vs_oracle(P, H, D):
    B, S = 2, 70 * P   # shards of 70 rows: ragged query and key tiles
    q, k, v = U.qkv(B, S, H, D, seed=P * 10 + H)
    out = _ring(P, q, k, v)
    assert not torch.isnan(out).any()
    U.assert_close(out, U.oracle_mha(q, k, v))
    assert torch.equal(out.view(torch.int16), _ring(P, q, k, v).view(torch.int16))   # deterministic


@pytest.mark.parametrize("dist", ["D1", "D4"])
def test_ring_peaky_and_local_distributions(dist):
    """Scores far apart between blocks exercise the lse weighting (one block dominates a row)."""
    P, B, S, H, D = 4, 1, 4 * 300, 3, 128
    q, k, v = U.qkv(B, S, H, D, seed=5, dist=dist)
    U.assert_close(_ring(P, q, k, v), U.oracle_mha(q, k, v))


def test_ring_closed_forms():
    P, B, S, H, D = 4, 1, 4 * 200, 2, 96
    q, k, v = U.qkv(B, S, H, D, dist="D2")   # Q = 0: mean of V over all S keys, across all ring blocks
    out = _ring(P, q, k, v).double().cpu()
    mean = v.double().cpu().mean(dim=1, keepdim=True).expand_as(out)
    assert (out - mean).abs().max().item() < 2e-3
    q, k, v = U.qkv(B, S, H, D, dist="D3")   # V = 1 -> 1
    assert (_ring(P, q, k, v).double().cpu() - 1).abs().max().item() <= 2 ** -7


def _usp(P, U, q, k, v):
    B, S, H, D = q.shape
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, ring=True, ulysses=U)
    qs, ks, vs = _shards(q, P), _shards(k, P), _shards(v, P)
    outs = [torch.full_like(t, float("nan")) for t in qs]
    ws = plan.workspace()
    spa.spa_ring_attention_local(plan, qs, ks, vs, outs, ws)
    torch.cuda.synchronize()
    return torch.cat(outs, dim=1)


@pytest.mark.parametrize("P,Ud,H,D", [(4, 2, 6, 128), (8, 2, 6, 96), (8, 4, 12, 64), (6, 3, 9, 128)])
def test_usp_hybrid_vs_oracle(P, Ud, H, D):
    """USP (Ulysses degree U x Ring degree P/U) through the C ABI: reshards inside Ulysses groups,
    ring attention across them; within tolerance of the oracle and deterministic."""
    B, S = 1, 64 * P
    q, k, v = U.qkv(B, S, H, D, seed=P * 10 + Ud)
    out = _usp(P, Ud, q, k, v)
    assert not torch.isnan(out).any()
    U.assert_close(out, U.oracle_mha(q, k, v))
    assert torch.equal(out.view(torch.int16), _usp(P, Ud, q, k, v).view(torch.int16))


@pytest.mark.parametrize("P,Ud", [(4, 1), (8, 1), (4, 2), (8, 4)])
def test_ring_and_usp_with_key_padding(P, Ud):
    """Key-padding masks on ring plans apply by global key position to every ring block (blocks wholly past
    kv_len contribute nothing: lse = -inf)."""
    B, S, H, D = 2, 96 * P, 2 * Ud, 96
    q, k, v = U.qkv(B, S, H, D, seed=P * 7 + Ud)
    kv_len = torch.tensor([S - 97, S // 3], dtype=torch.int32, device="cuda")
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, ring=True, ulysses=Ud)
    plan.set_kv_len(kv_len)
    qs, ks, vs = _shards(q, P), _shards(k, P), _shards(v, P)
    outs = [torch.full_like(t, float("nan")) for t in qs]
    spa.spa_ring_attention_local(plan, qs, ks, vs, outs, plan.workspace())
    torch.cuda.synchronize()
    Q, K, V = (t.detach().cpu().double().numpy() for t in (q, k, v))
    ref = oracle.mha_unsharded(Q, K, V, key_valid=oracle.key_valid_from_lengths(kv_len.tolist(), S))
    U.assert_close(torch.cat(outs, dim=1), ref)
