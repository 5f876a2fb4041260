"""Key-padding mask (Alg. 1 attention_mask; R20) and head padding
(R10) on the GPU, through the C ABI, vs the fp64 oracle (oracle.mha_unsharded
with key_valid / oracle.sp.padded_forward semantics) and bit-identity pins."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_12056_b200 import spa
from tests import gpu_util as U

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


def _oracle_masked(q, k, v, kv_len):
    Q, K, V = (t.detach().cpu().double().numpy() for t in (q, k, v))
    S = K.shape[1]
    return oracle.mha_unsharded(Q, K, V, key_valid=oracle.key_valid_from_lengths(kv_len, S))


def _i32(xs):
    return torch.tensor(xs, dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("D", [64, 96, 128])
def test_masked_attention_vs_oracle(D):
    """Prefix lengths: full, ragged inside a tile, exactly a tile boundary, one key, beyond S (clamped)."""
    B, S, H = 5, 700, 2
    q, k, v = U.qkv(B, S, H, D, seed=D)
    kv_len = [S, 301, 256, 1, 10_000]
    out = spa.attention(q, k, v, kv_len=_i32(kv_len))
    torch.cuda.synchronize()
    U.assert_close(out, _oracle_masked(q, k, v, [min(x, S) for x in kv_len]))


def test_zero_length_gives_zero_rows():
    B, S, H, D = 2, 300, 2, 128
    q, k, v = U.qkv(B, S, H, D, seed=4)
    out = spa.attention(q, k, v, kv_len=_i32([0, 300]))
    torch.cuda.synchronize()
    assert torch.count_nonzero(out[0]).item() == 0
    assert torch.equal(out[1].view(torch.int16), spa.attention(q[1:], k[1:], v[1:])[0].view(torch.int16))


@pytest.mark.parametrize("D", [96, 128])
def test_mask_equals_truncated_keys_bitwise_and_ignores_padding_values(D):
    """A prefix mask of length L is the unmasked kernel on K[:L], V[:L] (same tiles, same order), whatever
    the padded keys hold (here: huge scores and values)."""
    B, S, H, L = 1, 900, 3, 517
    q, k, v = U.qkv(B, S, H, D, seed=11)
    k2, v2 = k.clone(), v.clone()
    k2[:, L:] = 30.0
    v2[:, L:] = -1000.0
    out = spa.attention(q, k2, v2, kv_len=_i32([L]))
    ref = spa.attention(q, k[:, :L].contiguous(), v[:, :L].contiguous())
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


def _shards(x, n):
    S_l = x.shape[1] // n
    return [x[:, r * S_l:(r + 1) * S_l].contiguous() for r in range(n)]


def _sp(P, q, k, v, stages, kv_len=None, pad=False, ulysses=False):
    B, S, H, D = q.shape
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages, pad_heads=pad)
    if kv_len is not None:
        plan.set_kv_len(kv_len)
    qs, ks, vs = _shards(q, P), _shards(k, P), _shards(v, P)
    outs = [torch.full_like(t, float("nan")) for t in qs]
    ws = plan.workspace()
    (spa.spa_ulysses_attention_local if ulysses else spa.spa_pipesp_attention_local)(plan, qs, ks, vs, outs, ws)
    torch.cuda.synchronize()
    return torch.cat(outs, dim=1)


@pytest.mark.parametrize("P,stages", [(2, 1), (2, 4), (4, 2), (8, 24)])
def test_sp_key_padding_mask(P, stages):
    """Masked PipeSP over P virtual ranks: oracle tolerance, and the same bits as the masked single-GPU kernel."""
    B, S, H, D = 2, 96 * P, 24 if P == 8 else 4 * P, 128
    q, k, v = U.qkv(B, S, H, D, seed=P + stages)
    kv_len = _i32([S - 77, S // 3])
    single = spa.attention(q, k, v, kv_len=kv_len)
    out = _sp(P, q, k, v, stages, kv_len=kv_len)
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    U.assert_close(out, _oracle_masked(q, k, v, kv_len.tolist()))


@pytest.mark.parametrize("P,H,stages", [(4, 6, 1), (4, 6, 2), (3, 4, 2), (7, 24, 1), (7, 24, 4), (8, 20, 3)])
def test_sp_head_padding(P, H, stages):
    """H % P != 0 with pad_heads (24 heads on 7 GPUs -> 28): same bits as the single-GPU
    kernel on the real heads, within tolerance of the fp64 oracle; pad heads never touch the output."""
    B, D = 1, 96
    S = 40 * P
    q, k, v = U.qkv(B, S, H, D, seed=H * 10 + P)
    single = spa.attention(q, k, v)
    out = _sp(P, q, k, v, stages, pad=True)
    assert not torch.isnan(out).any()
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    U.assert_close(out, U.oracle_mha(q, k, v))
    uly = _sp(P, q, k, v, 1, pad=True, ulysses=True)
    assert torch.equal(uly.view(torch.int16), single.view(torch.int16))


def test_sp_padding_and_mask_together():
    P, B, S, H, D = 3, 2, 3 * 128, 4, 64
    q, k, v = U.qkv(B, S, H, D, seed=21)
    kv_len = _i32([200, 0])
    single = spa.attention(q, k, v, kv_len=kv_len)
    out = _sp(P, q, k, v, 2, kv_len=kv_len, pad=True)
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    assert torch.count_nonzero(out[1]).item() == 0
    U.assert_close(out, _oracle_masked(q, k, v, [200, 0]))
