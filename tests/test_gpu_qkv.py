"""GPU parity of the QKV projection fused with PipeSP (PAPER.md:155-157 projections,
PAPER.md:439 overlap with the input all-to-alls), through the C ABI.

* The tcgen05 projection GEMM against the fp64 oracle (oracle/projection.py): every element within the bound
  |gpu - exact| <= ulp_bf16(gpu)/2 + C * 2^-23 * sum_c |x_c w_c| (+ bias term) -- the bf16 output rounding plus
  an fp32-accumulation bound (R22); ragged M, N and K tails, batch > 1, D in {64, 96, 128}.
* The fused SP layer equals projection-then-attention BIT FOR BIT (spa_qkv_projection + the single-GPU kernel)
  at every rank count and stage split, and is within the attention tolerance of the oracle pipeline
  (bf16(X W^T + b) -> fp64 attention).
* Full size: HunyuanVideo-720p hidden states (C = 3072) over 8 virtual ranks, N_st = 3."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
from oracle import projection as pj
from paper_2511_12056_b200 import spa
from tests import gpu_util as U

pytestmark = pytest.mark.gpu


def _inputs(B, S, C, H, D, seed=0, device="cuda"):
    X = synthgen.gen_hidden_shard(seed, (B, S, C), 0, S, device=device)
    W = synthgen.gen_qkv_weight(seed, C, H, D, device=device)
    b = synthgen.gen_qkv_bias(seed, H, D, device=device)
    return X, W, b


def _check_projection(X, W, b, outs, H, D, rows=None):
    """Element bound vs the exact fp64 projection; returns the fraction equal to the oracle's bf16 rounding."""
    Xd = X.double().cpu().numpy()
    if rows is not None:
        Xd = Xd[:, rows]
    Wd = W.double().cpu().numpy()
    bd = None if b is None else b.double().cpu().numpy()
    exact = pj.qkv_projection(Xd, Wd, bd, H, D, round_bf16=False)
    ref = pj.qkv_projection(Xd, Wd, bd, H, D, round_bf16=True)
    C = Xd.shape[-1]
    absdot = np.abs(Xd).reshape(-1, C) @ np.abs(Wd).T                       # sum_c |x_c w_c|  [M, 3HD]
    if bd is not None:
        absdot = absdot + np.abs(bd)[None]
    bound_acc = (C + 1) * 2.0 ** -23 * absdot.reshape(Xd.shape[0], Xd.shape[1], 3, H, D)
    same = 0
    for t in range(3):
        g = outs[t] if rows is None else outs[t][:, rows]
        g = g.double().cpu().numpy()
        ulp = np.ldexp(1.0, np.frexp(np.abs(g))[1] - 8)
        err = np.abs(g - exact[t])
        assert np.all(err <= ulp / 2 + bound_acc[:, :, t] + 1e-30), float((err - ulp / 2 - bound_acc[:, :, t]).max())
        same += int((g == ref[t]).sum())
    return same / (3 * ref[0].size)


@pytest.mark.parametrize("B,S,C,H,D", [
    (1, 256, 256, 4, 64),     # one pair tile in M, N = 768 (3 column tiles)
    (2, 300, 200, 4, 96),     # ragged M (600 rows), N = 1152 (4.5 tiles), K tail (200 = 3*64 + 8)
    (1, 1000, 512, 2, 128),   # ragged M, N = 768
    (1, 4104, 384, 8, 128),   # many tiles: persistent loop over > 1 tile per pair
    (1, 100, 64, 1, 64),      # M < one CTA tile, N = 192 < one pair tile, K = one step
])
def test_projection_vs_oracle(B, S, C, H, D):
    X, W, b = _inputs(B, S, C, H, D)
    plan = spa.Plan(spa.Comm.loopback(1), B, S, H, D)
    wp = plan.pack_qkv_weight(W, b)
    q, k, v = (torch.empty((B, S, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(3))
    spa.spa_qkv_projection(plan, C, 0, X, wp, q, k, v)
    torch.cuda.synchronize()
    frac = _check_projection(X, W, b, (q, k, v), H, D)
    assert frac > 0.97, frac   # almost every element rounds like the exact value


def test_projection_without_bias_and_head_group_split():
    """bias = NULL; the packed layout of a 4-rank plan with 3 head groups: the standard-layout projection of every
    rank's shard is bit-identical to the 1-rank plan's (same K order per element)."""
    B, S, C, H, D, P = 1, 512, 256, 12, 64, 4
    X, W, _ = _inputs(B, S, C, H, D, seed=2)
    p1 = spa.Plan(spa.Comm.loopback(1), B, S, H, D)
    wp1 = p1.pack_qkv_weight(W, None)
    full = [torch.empty((B, S, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    spa.spa_qkv_projection(p1, C, 0, X, wp1, *full)
    torch.cuda.synchronize()
    _check_projection(X, W, None, full, H, D)
    pP = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=3)
    assert pP.stage_split == (3, 1, 1)
    wpP = pP.pack_qkv_weight(W, None)
    S_l = S // P
    for r in range(P):
        xr = X[:, r * S_l:(r + 1) * S_l].contiguous()
        outs = [torch.empty((B, S_l, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
        spa.spa_qkv_projection(pP, C, r, xr, wpP, *outs)
        torch.cuda.synchronize()
        for t in range(3):
            assert torch.equal(outs[t].view(torch.int16), full[t][:, r * S_l:(r + 1) * S_l].view(torch.int16))


def _fused(P, X, wp, C, H, D, stages, plan=None):
    B, S, _ = X.shape
    plan = plan or spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages)
    b = oracle.sp.shard_bounds(S, P)
    xs = [X[:, b[r]:b[r + 1]].contiguous() for r in range(P)]
    outs = [torch.empty((B, b[r + 1] - b[r], H, D), dtype=torch.bfloat16, device="cuda") for r in range(P)]
    ws = plan.qkv_workspace()
    spa.spa_pipesp_qkv_attention_local(plan, C, xs, wp, outs, ws)
    torch.cuda.synchronize()
    return torch.cat(outs, dim=1)


@pytest.mark.parametrize("P,stages,B,S,H,D,C", [
    (1, 1, 1, 384, 4, 64, 256), (1, 2, 2, 300, 4, 96, 256),
    (2, 1, 1, 512, 4, 64, 256), (2, 2, 1, 512, 4, 128, 512),
    (4, 1, 1, 1024, 8, 64, 512), (4, 2, 2, 1000, 8, 96, 384), (4, 4, 1, 1024, 8, 128, 1024),
    (8, 3, 1, 2048, 24, 64, 1536), (3, 2, 1, 1001, 6, 64, 384),
])
def test_fused_equals_projection_then_attention(P, stages, B, S, H, D, C):
    X, W, b = _inputs(B, S, C, H, D, seed=P + stages)
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages)
    wp = plan.pack_qkv_weight(W, b)
    out = _fused(P, X, wp, C, H, D, stages, plan)
    p1 = spa.Plan(spa.Comm.loopback(1), B, S, H, D)
    wp1 = p1.pack_qkv_weight(W, b)
    qkv = [torch.empty((B, S, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    spa.spa_qkv_projection(p1, C, 0, X, wp1, *qkv)
    single = spa.attention(*qkv)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    if S * H <= 8192:   # the whole oracle pipeline: bf16(X W^T + b) -> fp64 attention
        Q, K, V = pj.qkv_projection(X.double().cpu().numpy(), W.double().cpu().numpy(), b.double().cpu().numpy(), H, D)
        ref = oracle.mha_unsharded(Q, K, V)
        U.assert_close(out, ref)


def test_fused_skip_comm_and_profile():
    """Profile of a fused call: gemm launches = head groups x ranks, pack_ms = the projections."""
    P, B, S, H, D, C = 4, 1, 1024, 8, 64, 512
    X, W, b = _inputs(B, S, C, H, D, seed=9)
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=2)
    wp = plan.pack_qkv_weight(W, b)
    plan.set_option(spa.SPA_OPT_PROFILE, 1)
    plan.set_option(spa.SPA_OPT_COMM_SMS, 8)
    _fused(P, X, wp, C, H, D, 2, plan)
    prof = plan.last_profile()
    assert prof.gemm_launches == 2 * P and prof.n_stages == 2 and prof.pack_ms > 0


@pytest.mark.timeout(900)
def test_fullsize_720p_p8():
    """configs[3] with hidden states: S = 118,800, C = H*D = 3072, P = 8 virtual ranks, N_st = 3.  The fused layer is
    bit-identical to projection + the single-GPU kernel; the projection is checked on sampled rows against the fp64
    oracle, the attention output on sampled rows against the oracle applied to the GPU-projected Q, K, V."""
    w = synthgen.WORKLOADS["hy720p129f"]
    B, S, H, D, C, P = w.B, w.S, w.H, w.D, w.H * w.D, 8
    X, W, b = _inputs(B, S, C, H, D, seed=7)
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=3)
    wp = plan.pack_qkv_weight(W, b)
    out = _fused(P, X, wp, C, H, D, 3, plan)
    # the direct transport at full size: the projection GEMMs store into the owners (N_st = 3 and, with query chunks,
    # N_st = 24) -- the same bits
    for st in (3, 24):
        dp = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=st)
        dp.set_option(spa.SPA_OPT_DIRECT, 1)
        od = _fused(P, X, dp.pack_qkv_weight(W, b), C, H, D, st, dp)
        assert torch.equal(od.view(torch.int16), out.view(torch.int16)), st
        dp.close()
        del od
    del wp
    p1 = spa.Plan(spa.Comm.loopback(1), B, S, H, D)
    wp1 = p1.pack_qkv_weight(W, b)
    qkv = [torch.empty((B, S, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    spa.spa_qkv_projection(p1, C, 0, X, wp1, *qkv)
    single = spa.attention(*qkv)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), single.view(torch.int16))
    rng = np.random.default_rng(0)
    rows = torch.tensor(sorted(set(rng.integers(0, S, 192).tolist()) | {0, S - 1, S // 8, S // 8 - 1}))
    frac = _check_projection(X, W, b, qkv, H, D, rows=rows)
    assert frac > 0.97, frac
    q, k, v = qkv
    for h in (0, 11, 23):
        ref = oracle.attention_rows(q[0, rows, h].double().cpu().numpy(), k[0, :, h].double().cpu().numpy(),
                                    v[0, :, h].double().cpu().numpy())
        U.assert_close(out[0, rows, h], ref)


@pytest.mark.parametrize("P,stages,B,S,H,D,C", [
    (2, 1, 1, 512, 4, 64, 256), (2, 2, 2, 512, 4, 128, 512), (4, 2, 2, 1000, 8, 96, 384),
    (8, 3, 1, 2048, 24, 64, 1536), (3, 2, 1, 1001, 6, 64, 384), (4, 4, 1, 1024, 8, 128, 1024),
    (8, 24, 1, 2051, 24, 64, 1536), (3, 8, 2, 1001, 6, 96, 384), (2, 6, 1, 777, 2, 128, 256),   # query chunks
])
def test_fused_direct_equals_staged(P, stages, B, S, H, D, C):
    """Direct transport with the fused projections (SURVEY f1 + f3): each head group's GEMM stores its columns
    straight into every owner's receive regions (projection + pack + input all-to-all in one kernel) -- the same bits
    as the staged fused call, for uneven shards and B > 1 too."""
    X, W, b = _inputs(B, S, C, H, D, seed=17 + P + stages)
    staged = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages)
    wp = staged.pack_qkv_weight(W, b)
    ref = _fused(P, X, wp, C, H, D, stages, staged)
    direct = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages)
    direct.set_option(spa.SPA_OPT_DIRECT, 1)
    direct.set_option(spa.SPA_OPT_PROFILE, 1)
    out = _fused(P, X, wp, C, H, D, stages, direct)
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
    prof = direct.last_profile()
    G_h, n_chunks, _ = direct.stage_split
    assert prof.gemm_launches == G_h * P
    assert prof.copy_launches == 0   # the GEMMs moved every byte (query chunks too): no pack / exchange / unpack
