"""Sequence-parallel path on ONE GPU with P virtual ranks (loopback comm) through the C ABI:
reshard bit-exact vs the oracle permutation, PipeSP / Ulysses / Aco vs the fp64 oracle,
and bit-identity across rank counts and stage counts."""
import numpy as np
import pytest
import torch

import synthgen
from oracle import sp as osp
from paper_2511_12056_b200 import spa
from tests import gpu_util as U

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


def _shards(x, n):
    """sequence shards; uneven (first S % n ranks one token longer) when n does not divide S"""
    S = x.shape[1]
    out, t = [], 0
    for r in range(n):
        ln = S // n + (1 if r < S % n else 0)
        out.append(x[:, t:t + ln].contiguous())
        t += ln
    return out


def _u16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("D", [64, 96, 128])
def test_reshard_bit_exact(P, D):
    B, S, H = 2, 48 * P, 3 * P
    x = U.qkv(B, S, H, D, seed=P)[0]
    xs = _shards(x, P)
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=1)
    ws = plan.workspace()
    heads = [torch.empty(B, S, H // P, D, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
    spa.spa_reshard_seq_to_head_local(plan, xs, heads, ws)
    torch.cuda.synchronize()
    ref = osp.seq_to_head([_u16(t) for t in xs])
    for r in range(P):
        assert np.array_equal(_u16(heads[r]), ref[r]), r
    back = [torch.empty_like(t) for t in xs]
    spa.spa_reshard_head_to_seq_local(plan, heads, back, ws)
    torch.cuda.synchronize()
    ref_back = osp.head_to_seq(ref)
    for r in range(P):
        assert np.array_equal(_u16(back[r]), ref_back[r]) and torch.equal(back[r].view(torch.int16),
                                                                          xs[r].view(torch.int16))


def _pipesp(P, q, k, v, stages, ulysses=False, n_src=0):
    B, S, H, D = q.shape
    comm = spa.Comm.loopback(P)
    plan = spa.Plan(comm, B, S, H, D, stages=stages, n_src=n_src)
    n = n_src or P
    qs, ks, vs = _shards(q, n), _shards(k, n), _shards(v, n)
    outs = [torch.full_like(t, float("nan")) for t in qs]
    ws = plan.workspace()
    if n_src:
        spa.spa_aco_attention_local(plan, qs, ks, vs, outs, ws)
    elif ulysses:
        spa.spa_ulysses_attention_local(plan, qs, ks, vs, outs, ws)
    else:
        spa.spa_pipesp_attention_local(plan, qs, ks, vs, outs, ws)
    torch.cuda.synchronize()
    return torch.cat(outs, dim=1)


def test_tiny_config_p2_vs_oracle():
    """BASELINE configs[0]: B=1, S=256, H=4, D=64, P=2 virtual ranks, N_st in {1, 2}."""
    q, k, v = U.qkv(1, 256, 4, 64)
    ref = U.oracle_mha(q, k, v)
    for st in (1, 2):
        U.assert_close(_pipesp(2, q, k, v, st), ref)


@pytest.mark.parametrize("P,H,D,stages", [
    (2, 4, 128, 4), (4, 8, 96, 2), (4, 8, 96, 6), (8, 8, 64, 8), (8, 24, 128, 3), (8, 24, 128, 24),
    (8, 24, 96, 4), (4, 12, 64, 12),
])
def test_pipesp_vs_oracle_and_bit_identity(P, H, D, stages):
    B, S = 1, 64 * P + 0
    q, k, v = U.qkv(B, S, H, D, seed=P * 100 + stages)
    single = spa.attention(q, k, v)
    out = _pipesp(P, q, k, v, stages)
    U.assert_close(out, U.oracle_mha(q, k, v))
    # same bits as the single-GPU kernel: every row is computed independently of the split
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    uly = _pipesp(P, q, k, v, 1, ulysses=True)
    assert torch.equal(uly.view(torch.int16), single.view(torch.int16))


def test_ragged_sequence_and_batch():
    """S = 8 * 93 (tiles not multiples of 128), B = 2, all stage splits at P = 8, h = 3."""
    P, B, S, H, D = 8, 2, 8 * 93, 24, 128
    q, k, v = U.qkv(B, S, H, D, seed=7)
    single = spa.attention(q, k, v)
    U.assert_close(single, U.oracle_mha(q, k, v))
    for st in (1, 2, 3, 4, 6, 8, 12, 24):
        out = _pipesp(P, q, k, v, st)
        assert torch.equal(out.view(torch.int16), single.view(torch.int16)), st


@pytest.mark.parametrize("n_src,N,stages", [(6, 8, 1), (6, 8, 3), (3, 4, 2)])
def test_aco_loopback(n_src, N, stages):
    """Aco: heads over N owners, shards on n_src ranks; identical bits to the single-GPU result."""
    B, S, H, D = 1, 36 * n_src, 24, 128
    q, k, v = U.qkv(B, S, H, D, seed=n_src)
    single = spa.attention(q, k, v)
    out = _pipesp(N, q, k, v, stages, n_src=n_src)
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    U.assert_close(out, U.oracle_mha(q, k, v))


def test_profile_and_skip_comm():
    P, B, S, H, D = 4, 1, 1024, 8, 128
    q, k, v = U.qkv(B, S, H, D)
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=2)
    plan.set_option(spa.SPA_OPT_PROFILE, 1)
    qs, ks, vs = _shards(q, P), _shards(k, P), _shards(v, P)
    outs = [torch.empty_like(t) for t in qs]
    ws = plan.workspace()
    spa.spa_pipesp_attention_local(plan, qs, ks, vs, outs, ws)
    torch.cuda.synchronize()
    prof = plan.last_profile()
    assert prof.n_stages == 2 and prof.total_ms > 0 and prof.attn_ms[0] > 0 and prof.a2a_in_ms[1] > 0
    assert prof.attn_launches == 2 * P
    plan.set_option(spa.SPA_OPT_SKIP_COMM, 1)
    spa.spa_pipesp_attention_local(plan, qs, ks, vs, outs, ws)
    torch.cuda.synchronize()


def test_aco_busy_returns_busy():
    plan = spa.Plan(spa.Comm.loopback(8), 1, 96, 24, 64, stages=1, n_src=6)
    plan.set_option(spa.SPA_OPT_COPROC_BUSY, 1)
    x = torch.zeros(1, 16, 24, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(spa.SpaError) as e:
        spa.spa_aco_attention_local(plan, [x] * 6, [x] * 6, [x] * 6, [x] * 6, plan.workspace())
    assert e.value.status == 6


@pytest.mark.parametrize("P,S,stages", [(3, 3 * 100 + 2, 1), (3, 3 * 100 + 2, 3), (7, 7 * 64 + 5, 1), (8, 8 * 93 + 7, 6)])
def test_uneven_shards_bit_identical(P, S, stages):
    """S % P != 0 (R9): shards differ by one token; PipeSP and Ulysses still give the single-GPU bits."""
    B, D = 2, 96
    H = 3 * P
    q, k, v = U.qkv(B, S, H, D, seed=S)
    single = spa.attention(q, k, v)
    out = _pipesp(P, q, k, v, stages)
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    uly = _pipesp(P, q, k, v, 1, ulysses=True)
    assert torch.equal(uly.view(torch.int16), single.view(torch.int16))
    U.assert_close(out, U.oracle_mha(q, k, v))


@pytest.mark.parametrize("stages", [1, 3])
def test_aco_seven_plus_one(stages):
    """The paper's Aco example: H = 24 with 7 denoising GPUs, which Ulysses could only run with
    padding to 28 heads; with a decoding GPU as co-processor the 24 heads split 3 per owner over 8 GPUs and
    the sequence over 7 (unevenly)."""
    B, S, H, D = 1, 7 * 90 + 4, 24, 128
    q, k, v = U.qkv(B, S, H, D, seed=77)
    single = spa.attention(q, k, v)
    out = _pipesp(8, q, k, v, stages, n_src=7)
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    U.assert_close(out, U.oracle_mha(q, k, v))


def test_two_plans_on_two_streams_concurrently():
    """Stream semantics (include/spa.h): each call is ordered on the caller's stream; two plans driven from two
    streams at once (their comm streams, events and workspaces are separate) both give the single-GPU bits."""
    B, S, H, D = 1, 4 * 200, 8, 128
    q, k, v = U.qkv(B, S, H, D, seed=123)
    single = spa.attention(q, k, v)
    q2, k2, v2 = U.qkv(B, S, H, D, seed=321)
    single2 = spa.attention(q2, k2, v2)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    pa = spa.Plan(spa.Comm.loopback(4), B, S, H, D, stages=2)
    pb = spa.Plan(spa.Comm.loopback(4), B, S, H, D, stages=4)
    wa, wb = pa.workspace(), pb.workspace()
    outs_a = [torch.empty_like(t) for t in _shards(q, 4)]
    outs_b = [torch.empty_like(t) for t in _shards(q2, 4)]
    with torch.cuda.stream(s1):
        ia = [_shards(x, 4) for x in (q, k, v)]
    with torch.cuda.stream(s2):
        ib = [_shards(x, 4) for x in (q2, k2, v2)]
    torch.cuda.synchronize()
    for _ in range(3):
        spa.spa_pipesp_attention_local(pa, *ia, outs_a, wa, s1)
        spa.spa_pipesp_attention_local(pb, *ib, outs_b, wb, s2)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs_a, 1).view(torch.int16), single.view(torch.int16))
    assert torch.equal(torch.cat(outs_b, 1).view(torch.int16), single2.view(torch.int16))


@pytest.mark.parametrize("P,S,H,stages,pad,n_src,masked", [
    (2, 2 * 200, 4, 2, False, 0, False), (4, 4 * 150 + 3, 8, 4, False, 0, True), (8, 8 * 93, 24, 24, False, 0, False),
    (7, 7 * 64 + 5, 24, 1, True, 0, False), (8, 7 * 90 + 4, 24, 3, False, 7, False), (3, 3 * 100, 6, 6, False, 0, True),
])
def test_direct_transport_bit_identical(P, S, H, stages, pad, n_src, masked):
    """SPA_OPT_DIRECT (SURVEY f1 data path on loopback): pack into the owners' receive regions, attention epilogue
    into the sources' outputs -- same bits as the single-GPU kernel (and so as the staged exchange)."""
    B, D = 2, 128
    q, k, v = U.qkv(B, S, H, D, seed=S + P)
    kv_len = torch.tensor([S - 33, S // 2], dtype=torch.int32, device="cuda") if masked else None
    single = spa.attention(q, k, v, kv_len=kv_len)
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages, n_src=n_src, pad_heads=pad)
    plan.set_option(spa.SPA_OPT_DIRECT, 1)
    if masked:
        plan.set_kv_len(kv_len)
    n = n_src or P
    qs, ks, vs = _shards(q, n), _shards(k, n), _shards(v, n)
    outs = [torch.full_like(t, float("nan")) for t in qs]
    call = spa.spa_aco_attention_local if n_src else spa.spa_pipesp_attention_local
    call(plan, qs, ks, vs, outs, plan.workspace())
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs, dim=1).view(torch.int16), single.view(torch.int16))


def test_rank_only_measurement_mode():
    """SPA_OPT_RANK_ONLY (loopback): only virtual rank r's launches run -- 1 attention launch per stage instead of P,
    one pack and one unpack; SPA_OPT_LOOPBACK_CE moves the messages with copy engines (no copy-kernel launches)
    and leaves the result bits unchanged."""
    B, S, H, D, P = 1, 1024, 8, 64, 4
    q, k, v = (synthgen.gen_qkv_shard(0, t, (B, S, H, D), 0, S, device="cuda") for t in range(3))
    S_l = S // P
    shards = [[x[:, i * S_l:(i + 1) * S_l].contiguous() for i in range(P)] for x in (q, k, v)]
    outs = [torch.empty_like(t) for t in shards[0]]
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=2)
    ws = plan.workspace()
    plan.set_option(spa.SPA_OPT_PROFILE, 1)
    plan.set_option(spa.SPA_OPT_LOOPBACK_CE, 1)
    spa.spa_pipesp_attention_local(plan, *shards, outs, ws)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs, 1).view(torch.int16), spa.attention(q, k, v).view(torch.int16))
    assert plan.last_profile().copy_launches == 2   # pack + unpack kernels; the exchange ran on copy engines
    plan.set_option(spa.SPA_OPT_LOOPBACK_CE, 0)
    plan.set_option(spa.SPA_OPT_RANK_ONLY, 3)
    spa.spa_pipesp_attention_local(plan, *shards, outs, ws)
    torch.cuda.synchronize()
    prof = plan.last_profile()
    assert prof.attn_launches == 2 and prof.n_stages == 2


@pytest.mark.parametrize("P,stages,B,S,H,D,n_src,pad", [
    (2, 2, 1, 1024, 4, 64, 0, False), (4, 4, 2, 2048, 8, 128, 0, False), (4, 8, 1, 2051, 8, 96, 0, False),
    (8, 3, 1, 4096, 24, 128, 0, False), (8, 3, 1, 4096, 24, 64, 6, False), (3, 2, 1, 960, 4, 64, 0, True),
    (1, 4, 1, 1024, 8, 64, 0, False),
])
def test_hostbuf_sp_equals_device_call(P, stages, B, S, H, D, n_src, pad):
    """spa_pipesp_attention_hostbuf(_local): pinned host Q/K/V in, host O out, H2D / exchange / attention / D2H
    pipelined per head group -- the same bits as the single-GPU kernel (and so as the device-buffer SP call)."""
    q, k, v = (synthgen.gen_qkv_shard(3, t, (B, S, H, D), 0, S, device="cuda") for t in range(3))
    single = spa.attention(q, k, v)
    torch.cuda.synchronize()
    nsrc = n_src or P
    b = osp.shard_bounds(S, nsrc)
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages, n_src=n_src, pad_heads=pad)
    hs = [[x[:, b[r]:b[r + 1]].cpu().pin_memory() for r in range(nsrc)] for x in (q, k, v)]
    houts = [torch.zeros((B, b[r + 1] - b[r], H, D), dtype=torch.bfloat16).pin_memory() for r in range(nsrc)]
    ws = torch.empty(plan.host_sp_workspace_bytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):   # the same buffers twice (no state left behind)
        for o in houts:
            o.zero_()
        spa.spa_pipesp_attention_hostbuf_local(plan, *hs, houts, ws)
        torch.cuda.synchronize()
        assert torch.equal(torch.cat(houts, dim=1).view(torch.int16), single.cpu().view(torch.int16))


@pytest.mark.parametrize("window,direct", [(1, False), (4, False), (8, False), (4, True)])
def test_stage_window_bit_identical(window, direct):
    """SPA_OPT_STAGE_WINDOW: 1..8 stages in flight on as many compute streams -- the same bits as the single kernel."""
    B, S, H, D, P = 1, 2048, 24, 64, 8
    q, k, v = (synthgen.gen_qkv_shard(4, t, (B, S, H, D), 0, S, device="cuda") for t in range(3))
    single = spa.attention(q, k, v)
    S_l = S // P
    shards = [[x[:, i * S_l:(i + 1) * S_l].contiguous() for i in range(P)] for x in (q, k, v)]
    outs = [torch.empty_like(t) for t in shards[0]]
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=24)
    plan.set_option(spa.SPA_OPT_STAGE_WINDOW, window)
    if direct:
        plan.set_option(spa.SPA_OPT_DIRECT, 1)
    spa.spa_pipesp_attention_local(plan, *shards, outs, plan.workspace())
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs, 1).view(torch.int16), single.view(torch.int16))
