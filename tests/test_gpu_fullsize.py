"""Full-size parity at the BASELINE.json shapes, in the launch configurations bench.py times.

Per (config, value distribution) one test: the inputs are generated at full size, every path that
serves the config runs on them, and the outputs are compared with the fp64 oracle on >= 1024 sampled
query rows x 6 heads spread over H (SURVEY.md §8(c) "Sampled rows at scale").  Each output row depends
only on its own query row and the full K/V of its head (Alg. 1 l.3), so a sampled row is
an exact check.  The sample holds uniform random rows plus every shard-edge row for P in {6, 7, 8}
(including the uneven 7-way shards of Aco 7+1), the query-chunk edges of N_st = 24, and the 16 rows of
the ragged last 128-row tile of 720p.

Paths: the single-GPU kernel and the 1-rank plan call (the N=1 bench configuration), PipeSP over P = 8
virtual ranks with N_st in {1, 3, 24} (+ the direct transport at N_st = 3), Aco 6+2 and the paper's 7+1
 at 720p, Ring-Attention over 8 ranks at OSP, and a key-padding mask at HY-544p.  The
bit-identity of every staged path with the single kernel (R18) is asserted on the whole tensor.

Worst max-abs / rel-L2 per (config, distribution, path) are printed and, when SPA_PARITY_LOG names a
file, appended to it as JSON lines (profiles/r02/parity_fullsize.jsonl)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synthgen
from paper_2511_12056_b200 import spa
from tests import gpu_util as U

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1800)]

HEADS = [0, 5, 9, 14, 18, 23]      # 6 heads spread over H = 24
N_RANDOM = 1024


def _gen(w, dist, seed):
    return [synthgen.gen_qkv_shard(seed, t, (w.B, w.S, w.H, w.D), 0, w.S, dist=dist, device="cuda")
            for t in range(3)]


def _bounds(S, P):
    """Shard starts of P source ranks, lengths differing by <= 1 (R9)."""
    lens = [S // P + (1 if r < S % P else 0) for r in range(P)]
    return np.concatenate([[0], np.cumsum(lens)]).tolist()


def sample_rows(S, seed=0):
    rng = np.random.default_rng(seed)
    rows = set(rng.integers(0, S, N_RANDOM).tolist())
    for P in (6, 7, 8):
        b = _bounds(S, P)
        for r in range(P):
            rows.update((b[r], b[r + 1] - 1))
            if P == 8:   # query-chunk edges of N_st = 24 at P = 8 (C = 8 chunks per head, R7)
                L = b[r + 1] - b[r]
                rows.update(b[r] + c * L // 8 for c in range(8))
                rows.update(b[r] + (c + 1) * L // 8 - 1 for c in range(8))
    rows.update(range((S // 128) * 128, S))   # the ragged last tile (16 rows at 720p)
    return torch.tensor(sorted(rows))


class Ref:
    """fp64 oracle rows for the sampled (row, head) pairs of one input set."""

    def __init__(self, q, k, v, rows, heads, kv_len=None):
        self.rows, self.heads = rows, heads
        ref = []
        for h in heads:
            L = q.shape[1] if kv_len is None else kv_len
            Q = q[0, rows, h].double().cpu().numpy()
            K = k[0, :L, h].double().cpu().numpy()
            V = v[0, :L, h].double().cpu().numpy()
            ref.append(oracle.attention_rows(Q, K, V))
        self.ref = np.stack(ref)

    def errors(self, out):
        got = np.stack([out[0, self.rows, h].double().cpu().numpy() for h in self.heads])
        d = got - self.ref
        return (float(np.abs(d).max()), float(np.linalg.norm(d) / np.linalg.norm(self.ref)),
                float(np.abs(self.ref).max()))


def _log(config, dist, path, err, n_pairs):
    ma, rl, refmax = err
    rec = {"config": config, "dist": dist, "path": path, "max_abs": ma, "rel_l2": rl, "ref_max_abs": refmax,
           "max_abs_over_ref_max": ma / refmax, "pairs": n_pairs, "tol": {"max_abs": U.MAX_ABS, "rel_l2": U.REL_L2}}
    print(json.dumps(rec))
    dst = os.environ.get("SPA_PARITY_LOG")
    if dst:
        with open(dst, "a") as f:
            f.write(json.dumps(rec) + "\n")
    assert ma <= U.MAX_ABS and rl <= U.REL_L2, rec


def _same(a, b):
    return torch.equal(a.view(torch.int16), b.view(torch.int16))


def _shards(x, bounds):
    return [x[:, bounds[r]:bounds[r + 1]].contiguous() for r in range(len(bounds) - 1)]


def _sp(P, q, k, v, stages, n_src=0, direct=False, ring=False, kv_len=None):
    B, S, H, D = q.shape
    plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages, n_src=n_src, ring=ring)
    if direct:
        plan.set_option(spa.SPA_OPT_DIRECT, 1)
    if kv_len is not None:
        plan.set_kv_len(kv_len)
    b = _bounds(S, n_src or P)
    qs, ks, vs = (_shards(x, b) for x in (q, k, v))
    outs = [torch.empty_like(t) for t in qs]
    ws = plan.workspace()
    call = spa.spa_ring_attention_local if ring else (
        spa.spa_aco_attention_local if n_src else spa.spa_pipesp_attention_local)
    call(plan, qs, ks, vs, outs, ws)
    torch.cuda.synchronize()
    del ws, qs, ks, vs
    plan.close()
    return torch.cat(outs, dim=1)


CASES = [(c, d) for c in ("osp480p93f", "hy544p129f", "hy720p129f") for d in ("D0", "D1", "D4")]


@pytest.mark.parametrize("config,dist", CASES)
def test_fullsize_sampled_rows(config, dist):
    w = synthgen.WORKLOADS[config]
    seed = {"D0": 0, "D1": 1, "D4": 4}[dist]
    q, k, v = _gen(w, dist, seed)
    rows = sample_rows(w.S, seed)
    assert len(rows) >= N_RANDOM
    ref = Ref(q, k, v, rows, HEADS)
    npairs = len(rows) * len(HEADS)

    single = spa.attention(q, k, v)
    torch.cuda.synchronize()
    assert not torch.isnan(single.float()).any()
    _log(config, dist, "single_kernel", ref.errors(single), npairs)

    # the N=1 bench configuration: a 1-rank plan call on all heads
    plan = spa.Plan(spa.Comm.loopback(1), w.B, w.S, w.H, w.D)
    out1 = torch.empty_like(q)
    spa.spa_pipesp_attention_local(plan, [q], [k], [v], [out1], plan.workspace())
    torch.cuda.synchronize()
    assert _same(out1, single)
    _log(config, dist, "plan_P1", ref.errors(out1), npairs)
    del out1

    for st in (1, 3, 24):   # PipeSP over 8 virtual ranks; N_st = 1 is Ulysses
        out = _sp(8, q, k, v, st)
        assert _same(out, single), st
        _log(config, dist, f"pipesp_P8_Nst{st}", ref.errors(out), npairs)
        del out
    out = _sp(8, q, k, v, 3, direct=True)     # SPA_OPT_DIRECT data path (loopback model)
    assert _same(out, single)
    del out

    if config == "hy720p129f":                 # Aco: configs[4] 6+2, and the paper's 7+1 (uneven shards)
        for n_src in (6, 7):
            out = _sp(8, q, k, v, 3, n_src=n_src)
            assert _same(out, single), n_src
            _log(config, dist, f"aco_{n_src}+{8 - n_src}", ref.errors(out), npairs)
            del out
    if config == "osp480p93f":                 # Ring-Attention over 8 ranks (R21): a different summation order
        out = _sp(8, q, k, v, 1, ring=True)
        _log(config, dist, "ring_P8", ref.errors(out), npairs)
        del out
    if config == "hy544p129f":                 # key-padding mask (R20): 70,001 of 76,032 keys valid
        L = 70_001
        kv_len = torch.tensor([L], dtype=torch.int32, device="cuda")
        masked = spa.attention(q, k, v, kv_len=kv_len)
        torch.cuda.synchronize()
        mref = Ref(q, k, v, rows, HEADS, kv_len=L)
        _log(config, dist, "masked_single", mref.errors(masked), npairs)
        out = _sp(4, q, k, v, 2, kv_len=kv_len)
        assert _same(out, masked)
        _log(config, dist, "masked_pipesp_P4_Nst2", mref.errors(out), npairs)


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
