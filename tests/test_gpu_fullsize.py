"""Full-size parity at the BASELINE.json shapes, in the launch configuration bench.py times:
sampled output rows against the fp64 oracle (each output row depends only on its own query row
and the full K/V of its head, so a sampled row is an exact check), edge rows included
(first/last token of every rank shard, the ragged tail of 720p), plus properties at full size."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
from paper_2511_12056_b200 import spa
from tests import gpu_util as U

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1200)]


def _gen(B, S, H, D, seed=0):
    return [synthgen.gen_qkv_shard(seed, t, (B, S, H, D), 0, S, device="cuda") for t in range(3)]


def _check_rows(q, k, v, out, rows, heads, b=0):
    """oracle on the sampled (row, head) pairs; returns (max_abs, rel_l2) over all of them."""
    got, ref = [], []
    for h in heads:
        Q = q[b, rows, h].double().cpu().numpy()
        K = k[b, :, h].double().cpu().numpy()
        V = v[b, :, h].double().cpu().numpy()
        ref.append(oracle.attention_rows(Q, K, V))
        got.append(out[b, rows, h].double().cpu().numpy())
    got, ref = np.stack(got), np.stack(ref)
    d = got - ref
    return float(np.abs(d).max()), float(np.linalg.norm(d) / np.linalg.norm(ref))


def _sample(S, P, n=48, seed=0):
    rng = np.random.default_rng(seed)
    S_l = S // P
    edges = [x for r in range(P) for x in (r * S_l, r * S_l + S_l - 1)]
    tail = list(range((S // 128) * 128, S)) if S % 128 else []
    rows = sorted(set(rng.integers(0, S, n).tolist() + edges + tail[:16]))
    return torch.tensor(rows)


def _pipesp(P, q, k, v, stages, direct=False):
    B, S, H, D = q.shape
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages)
    if direct:
        plan.set_option(spa.SPA_OPT_DIRECT, 1)
    S_l = S // P
    shards = [[x[:, r * S_l:(r + 1) * S_l].contiguous() for r in range(P)] for x in (q, k, v)]
    outs = [torch.empty_like(t) for t in shards[0]]
    ws = plan.workspace()
    spa.spa_pipesp_attention_local(plan, *shards, outs, ws)
    torch.cuda.synchronize()
    del ws
    return torch.cat(outs, dim=1)


@pytest.mark.parametrize("name", ["osp480p93f", "hy544p129f"])
def test_single_gpu_baseline_configs(name):
    """configs[1] / configs[2] at P=1 (the N=1 bench configuration: one plan call on all heads)."""
    w = synthgen.WORKLOADS[name]
    q, k, v = _gen(w.B, w.S, w.H, w.D)
    out = torch.empty_like(q)
    plan = spa.Plan(spa.Comm.loopback(1), w.B, w.S, w.H, w.D)
    spa.spa_pipesp_attention_local(plan, [q], [k], [v], [out], plan.workspace())
    torch.cuda.synchronize()
    assert not torch.isnan(out.float()).any()
    ma, rl = _check_rows(q, k, v, out, _sample(w.S, 1), heads=[0, w.H // 2, w.H - 1])
    assert ma <= U.MAX_ABS and rl <= U.REL_L2, (ma, rl)


def test_720p_p8_pipesp_stages_bit_identical():
    """configs[3]: 720p x 129f (S = 118,800, ragged tail of 16 rows), P = 8 virtual ranks, N_st in {1, 3, 24}:
    sampled rows vs the oracle, and every stage split bit-identical to the single-GPU kernel."""
    w = synthgen.WORKLOADS["hy720p129f"]
    q, k, v = _gen(w.B, w.S, w.H, w.D)
    single = spa.attention(q, k, v)
    torch.cuda.synchronize()
    ma, rl = _check_rows(q, k, v, single, _sample(w.S, 8, n=32), heads=[0, 23])
    assert ma <= U.MAX_ABS and rl <= U.REL_L2, (ma, rl)
    for st in (1, 3, 24):
        out = _pipesp(8, q, k, v, st)
        assert torch.equal(out.view(torch.int16), single.view(torch.int16)), st
        del out
    out = _pipesp(8, q, k, v, 3, direct=True)   # SPA_OPT_DIRECT: the f1 data path (loopback model)
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))


def test_aco_720p_6_plus_2():
    """configs[4]: Aco, shards on 6 denoising ranks, heads over 6+2 owners, S = 118,800."""
    w = synthgen.WORKLOADS["hy720p129f"]
    q, k, v = _gen(w.B, w.S, w.H, w.D, seed=1)
    single = spa.attention(q, k, v)
    plan = spa.Plan(spa.Comm.loopback(8), w.B, w.S, w.H, w.D, stages=3, n_src=6)
    S_l = w.S // 6
    shards = [[x[:, r * S_l:(r + 1) * S_l].contiguous() for r in range(6)] for x in (q, k, v)]
    outs = [torch.empty_like(t) for t in shards[0]]
    spa.spa_aco_attention_local(plan, *shards, outs, plan.workspace())
    torch.cuda.synchronize()
    out = torch.cat(outs, dim=1)
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    ma, rl = _check_rows(q, k, v, out, _sample(w.S, 6, n=24, seed=3), heads=[5])
    assert ma <= U.MAX_ABS and rl <= U.REL_L2, (ma, rl)


def test_fullsize_closed_forms():
    """Properties that hold at any size: V == 1 -> O == 1; Q == 0 -> O = column mean of V."""
    B, S, H, D = 1, 28_800, 4, 96
    q, k, v = (synthgen.gen_qkv_shard(0, t, (B, S, H, D), 0, S, dist="D3", device="cuda") for t in range(3))
    out = spa.attention(q, k, v).float()
    assert (out - 1).abs().max().item() <= 2 ** -7
    q, k, v = (synthgen.gen_qkv_shard(0, t, (B, S, H, D), 0, S, dist="D2", device="cuda") for t in range(3))
    out = spa.attention(q, k, v).double()
    mean = v.double().mean(dim=1, keepdim=True)
    assert (out - mean).abs().max().item() < 1e-3


def test_ring_osp_p8_fullsize():
    """Ring-Attention (R21) at configs[1] size over 8 virtual ranks: sampled rows vs the oracle."""
    w = synthgen.WORKLOADS["osp480p93f"]
    q, k, v = _gen(w.B, w.S, w.H, w.D, seed=2)
    P = 8
    plan = spa.Plan(spa.Comm.loopback(P), w.B, w.S, w.H, w.D, ring=True)
    S_l = w.S // P
    shards = [[x[:, r * S_l:(r + 1) * S_l].contiguous() for r in range(P)] for x in (q, k, v)]
    outs = [torch.empty_like(t) for t in shards[0]]
    ws = plan.workspace()
    spa.spa_ring_attention_local(plan, *shards, outs, ws)
    torch.cuda.synchronize()
    del ws
    out = torch.cat(outs, dim=1)
    ma, rl = _check_rows(q, k, v, out, _sample(w.S, P, n=32, seed=4), heads=[0, 23])
    assert ma <= U.MAX_ABS and rl <= U.REL_L2, (ma, rl)


def test_key_padding_mask_fullsize():
    """Key-padding mask (R20) at configs[2] size: kv_len = 70,001 of 76,032 keys, sampled rows vs the oracle on
    the truncated keys, and the masked PipeSP at P = 4 bit-identical to the masked single-GPU kernel."""
    w = synthgen.WORKLOADS["hy544p129f"]
    q, k, v = _gen(w.B, w.S, w.H, w.D, seed=3)
    L = 70_001
    kv_len = torch.tensor([L], dtype=torch.int32, device="cuda")
    single = spa.attention(q, k, v, kv_len=kv_len)
    torch.cuda.synchronize()
    ma, rl = _check_rows(q, k[:, :L], v[:, :L], single, _sample(w.S, 4, n=24, seed=5), heads=[7])
    assert ma <= U.MAX_ABS and rl <= U.REL_L2, (ma, rl)
    P = 4
    plan = spa.Plan(spa.Comm.loopback(P), w.B, w.S, w.H, w.D, stages=2)
    plan.set_kv_len(kv_len)
    S_l = w.S // P
    shards = [[x[:, r * S_l:(r + 1) * S_l].contiguous() for r in range(P)] for x in (q, k, v)]
    outs = [torch.empty_like(t) for t in shards[0]]
    ws = plan.workspace()
    spa.spa_pipesp_attention_local(plan, *shards, outs, ws)
    torch.cuda.synchronize()
    del ws
    assert torch.equal(torch.cat(outs, dim=1).view(torch.int16), single.view(torch.int16))


def test_aco_720p_seven_plus_one():
    """The paper's Aco example at configs[3] size: S = 118,800 over 7 denoising ranks (uneven:
    16,972 / 16,971 tokens), 24 heads over 7 + 1 owners; bit-identical to the single-GPU kernel."""
    w = synthgen.WORKLOADS["hy720p129f"]
    q, k, v = _gen(w.B, w.S, w.H, w.D, seed=4)
    single = spa.attention(q, k, v)
    plan = spa.Plan(spa.Comm.loopback(8), w.B, w.S, w.H, w.D, stages=3, n_src=7)
    shards, t = [[], [], []], 0
    for r in range(7):
        ln = w.S // 7 + (1 if r < w.S % 7 else 0)
        for i, x in enumerate((q, k, v)):
            shards[i].append(x[:, t:t + ln].contiguous())
        t += ln
    outs = [torch.empty_like(x) for x in shards[0]]
    ws = plan.workspace()
    spa.spa_aco_attention_local(plan, *shards, outs, ws)
    torch.cuda.synchronize()
    del ws
    out = torch.cat(outs, dim=1)
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    ma, rl = _check_rows(q, k, v, out, _sample(w.S, 7, n=16, seed=6), heads=[21])
    assert ma <= U.MAX_ABS and rl <= U.REL_L2, (ma, rl)
