"""CPU emulation of the library's multi-rank HOST logic (test helper, no GPU).

Executes, on numpy byte buffers, exactly what a plan describes through the C ABI:
the pack copy jobs, each stage's message list (matched per ordered rank pair, NCCL
semantics), a stand-in for the attention kernel, and the unpack (Psi_g) jobs.
With the identity stand-in (O := Q) the output must equal the input: this checks
every offset, stride and message of the plan -- the part of the NCCL path that a
single-GPU box cannot exercise -- against the paper's reshard semantics.
"""
from __future__ import annotations

import numpy as np

from paper_2511_12056_b200 import spa


def run_copy(desc, bufs_src: np.ndarray, bufs_dst: np.ndarray):
    c = list(desc.count)
    ss, ds = list(desc.src_stride), list(desc.dst_stride)
    rb = desc.run_bytes
    for i3 in range(c[0]):
        for i2 in range(c[1]):
            for i1 in range(c[2]):
                for i0 in range(c[3]):
                    so = desc.src_off + i3 * ss[0] + i2 * ss[1] + i1 * ss[2] + i0 * ss[3]
                    do = desc.dst_off + i3 * ds[0] + i2 * ds[1] + i1 * ds[2] + i0 * ds[3]
                    bufs_dst[do:do + rb] = bufs_src[so:so + rb]


def exchange(plans, stage: int, direction: int, ws):
    """plans[r] = Plan on a host comm of rank r; ws[r] = that rank's workspace bytes."""
    P = len(plans)
    msgs = [plans[r].describe_messages(stage, direction, r) for r in range(P)]
    for src in range(P):
        for dst in range(P):
            sends = [m for m in msgs[src] if not m.is_recv and m.peer == dst]
            recvs = [m for m in msgs[dst] if m.is_recv and m.peer == src]
            assert len(sends) == len(recvs), (src, dst, len(sends), len(recvs))
            for s, r in zip(sends, recvs):
                assert s.bytes == r.bytes and s.buf == r.buf == spa.BUF_WS
                ws[dst][r.off:r.off + r.bytes] = ws[src][s.off:s.off + s.bytes]


def identity_attention(plan, stage: int, rank: int, wsr: np.ndarray):
    """O := Q for the stage's query rows (checks the attention descriptor's Q/O regions)."""
    a = plan.describe_attention(stage, rank)
    n = a.B * a.Sq * a.q_tok_stride * 2   # whole token rows of the group (pad-head slots included)
    wsr[a.o_off:a.o_off + n] = wsr[a.q_off:a.q_off + n]
    # K/V regions must hold full sequences of the stage's heads: touch-check the extents
    kv = a.B * a.Skv * a.kv_tok_stride * 2
    assert a.k_off + kv <= len(wsr) and a.v_off + kv <= len(wsr)


def run_path(plans, xs_q, xs_k, xs_v, attn=identity_attention):
    """Full per-rank path on host buffers. xs_*: list (per source rank) of uint8 arrays."""
    P = len(plans)
    nbytes = plans[0].workspace_bytes
    ws = [np.zeros(nbytes, dtype=np.uint8) for _ in range(P)]
    n_src = plans[0].n_src
    outs = [np.zeros_like(xs_q[r]) for r in range(n_src)]
    for r in range(n_src):
        user = {spa.BUF_Q: xs_q[r], spa.BUF_K: xs_k[r], spa.BUF_V: xs_v[r]}
        for d in plans[r].describe_pack(r):
            run_copy(d, user[d.src_buf], ws[r])
    G_h, C, g = plans[0].stage_split
    for k in range(G_h * C):
        exchange(plans, k, 0, ws)
        for r in range(P):
            attn(plans[r], k, r, ws[r])
        exchange(plans, k, 1, ws)
    for r in range(n_src):
        for d in plans[r].describe_unpack(r):
            run_copy(d, ws[r], outs[r])
    return outs
