"""Multi-process check of the library's NCCL-path host logic over gloo (CPU, world_size 2).

Each process plays one rank: it builds the plan on a host-only comm (same plan as the NCCL path),
runs the described pack jobs, exchanges exactly the described per-stage messages with the other
process through torch.distributed (gloo) point-to-point, applies an identity "attention" to the
described regions, runs the output exchange and the described unpack (Psi_g).  The output must
equal the input element for element, for every stage split, for Aco (1 source + 1 co-processor) and
for head padding (H odd), and the ring plan's described K/V rotation (R21).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(plan, stage, direction, rank, ws):
    from paper_2511_12056_b200 import spa
    msgs = plan.describe_messages(stage, direction, rank)
    reqs, counters = [], {}
    recv_bufs = []
    for m in msgs:
        assert m.buf == spa.BUF_WS
        key = (m.peer, m.is_recv)
        tag = counters.get(key, 0)
        counters[key] = tag + 1
        if m.peer == rank:
            continue
        if m.is_recv:
            t = torch.empty(m.bytes, dtype=torch.uint8)
            reqs.append(dist.irecv(t, src=m.peer, tag=tag))
            recv_bufs.append((t, m.off))
        else:
            reqs.append(dist.isend(torch.from_numpy(ws[m.off:m.off + m.bytes].copy()), dst=m.peer, tag=tag))
    # self messages: i-th send to self matches i-th receive from self
    sends = [m for m in msgs if m.peer == rank and not m.is_recv]
    recvs = [m for m in msgs if m.peer == rank and m.is_recv]
    assert len(sends) == len(recvs)
    for s, r in zip(sends, recvs):
        ws[r.off:r.off + r.bytes] = ws[s.off:s.off + s.bytes]
    for q in reqs:
        q.wait()
    for t, off in recv_bufs:
        ws[off:off + t.numel()] = t.numpy()


def _worker(rank, world, port, cases, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_12056_b200 import spa
    from tests import hostsim
    ok = True
    for (B, S, H, D, stages, n_src, pad) in cases:
        plan = spa.Plan(spa.Comm.host(world, rank), B, S, H, D, stages=stages, n_src=n_src, pad_heads=pad)
        nsrc = n_src or world
        bnd = [0]
        for r in range(nsrc):   # uneven shards when nsrc does not divide S (first S % nsrc ranks longer)
            bnd.append(bnd[-1] + S // nsrc + (1 if r < S % nsrc else 0))
        X = ((np.arange(B * S * H * D) * 2654435761) % 65521).astype(np.uint16).reshape(B, S, H, D)
        ws = np.zeros(plan.workspace_bytes, dtype=np.uint8)
        x = None
        if rank < nsrc:
            x = np.ascontiguousarray(X[:, bnd[rank]:bnd[rank + 1]]).view(np.uint8).reshape(-1)
            for d in plan.describe_pack(rank):
                hostsim.run_copy(d, x, ws)
        G_h, C, g = plan.stage_split
        for k in range(G_h * C):
            _exchange(plan, k, 0, rank, ws)
            hostsim.identity_attention(plan, k, rank, ws)
            _exchange(plan, k, 1, rank, ws)
        if rank < nsrc:
            out = np.zeros_like(x)
            for d in plan.describe_unpack(rank):
                hostsim.run_copy(d, ws, out)
            ok &= bool(np.array_equal(out, x))
        plan.close()
    # ring plan (R21): the described K/V messages of every step, exchanged for real over gloo; after step t the
    # receive slot holds the blocks of rank (rank - t - 1) mod P
    B, S, H, D = 1, 2 * 32, 3, 64
    plan = spa.Plan(spa.Comm.host(world, rank), B, S, H, D, ring=True)
    blk = B * (S // world) * H * D * 2
    K = np.full(blk, 10 + rank, dtype=np.uint8)
    V = np.full(blk, 20 + rank, dtype=np.uint8)
    ws = np.zeros(plan.workspace_bytes, dtype=np.uint8)
    for t in range(world - 1):
        msgs = plan.describe_ring(t, rank)
        reqs, rbufs = [], []
        for i, m in enumerate(msgs):
            if m.is_recv:
                buf = torch.empty(m.bytes, dtype=torch.uint8)
                reqs.append(dist.irecv(buf, src=m.peer, tag=100 * t + i - 2))
                rbufs.append((buf, m.off))
            else:
                src = K if m.buf == spa.BUF_K else V if m.buf == spa.BUF_V else ws[m.off:m.off + m.bytes]
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(src)), dst=m.peer, tag=100 * t + i))
        for q in reqs:
            q.wait()
        for buf, off in rbufs:
            ws[off:off + buf.numel()] = buf.numpy()
        owner = (rank - t - 1) % world
        k_off, v_off = [m.off for m in msgs if m.is_recv]
        ok &= bool((ws[k_off:k_off + blk] == 10 + owner).all() and (ws[v_off:v_off + blk] == 20 + owner).all())
    plan.close()
    result[rank] = int(ok)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_process_gloo_exchange():
    # (B, S, H, D, stages, n_src, pad_heads); the last two: H odd over 2 ranks with head padding
    cases = [(1, 64, 4, 64, 1, 0, 0), (1, 64, 4, 64, 2, 0, 0), (2, 64, 4, 96, 4, 0, 0), (1, 128, 8, 128, 8, 0, 0),
             (1, 96, 6, 64, 6, 0, 0), (1, 48, 2, 64, 1, 1, 0), (2, 48, 4, 64, 2, 1, 0), (1, 64, 3, 64, 2, 0, 1),
             (2, 64, 5, 96, 3, 0, 1), (1, 63, 4, 64, 2, 0, 0), (2, 63, 6, 64, 3, 1, 0)]
    world = 2
    ctx = mp.get_context("spawn")
    result = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, result)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert list(result) == [1] * world
