"""The P2P transport (spa_comm_init_p2p) with REAL processes: P processes share cuda:0, each
maps the others' workspaces through CUDA IPC and the exchange is ordered by cross-process epoch flags
(cuStreamWriteValue32 / cuStreamWaitValue32).  Apart from where the peer memory physically sits (the same HBM here,
another GPU over NVLink in production), this is the multi-GPU code path: separate CUDA contexts, separate streams,
peer pointers, no shared host state.  Every rank's output must equal the single-GPU kernel bit for bit, on every
call of the same plan (the epochs advance), for the staged copy-engine exchange and the direct (kernel-store)
transport, PipeSP / Ulysses / Aco / the fused QKV projection, and Ring-Attention / USP (bit-identical to the same
plan over virtual ranks on one GPU)."""
import socket

import pytest
import torch.multiprocessing as mp

from tests import p2p_worker

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(world, case):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    procs = [ctx.Process(target=p2p_worker.run, args=(r, world, _port_cache[0], case, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    alive = [p for p in procs if p.is_alive()]
    for p in alive:
        p.kill()
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not alive, f"{len(alive)} rank(s) hung"
    assert not errs, errs[0][1]
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


_port_cache = [0]


@pytest.mark.parametrize("world,case", [
    (2, dict(B=1, S=2048, H=4, D=128, stages=1)),
    (2, dict(B=2, S=1000, H=4, D=64, stages=2)),
    (4, dict(B=1, S=4096, H=8, D=128, stages=4)),
    (4, dict(B=1, S=4099, H=8, D=96, stages=2)),                 # uneven shards (R9)
    (4, dict(B=1, S=4096, H=8, D=128, stages=8)),                 # query chunks (C = 4)
    (2, dict(B=1, S=2048, H=4, D=128, stages=2, ulysses=True)),
    (2, dict(B=1, S=2048, H=4, D=128, stages=2, direct=True)),
    (4, dict(B=1, S=4096, H=8, D=64, stages=4, direct=True)),
    (4, dict(B=1, S=3000, H=8, D=128, stages=2, n_src=3)),        # Aco 3 + 1
    (4, dict(B=1, S=3000, H=8, D=128, stages=2, n_src=3, direct=True)),
    (2, dict(B=1, S=2048, H=4, D=128, stages=2, qkv=True)),       # f3 over the P2P transport
    (2, dict(B=1, S=2048, H=4, D=128, stages=2, qkv=True, direct=True)),   # projection GEMM stores into the peers
    (4, dict(B=2, S=3001, H=8, D=64, stages=2, qkv=True, direct=True)),
    (4, dict(B=1, S=4099, H=8, D=128, stages=8, qkv=True, direct=True)),   # + query chunks (C = 4)
    (8, dict(B=1, S=8192, H=24, D=128, stages=3)),
    (2, dict(B=1, S=2048, H=3, D=128, ring=True)),                # Ring-Attention over P2P (R21, any H)
    (4, dict(B=2, S=4096, H=5, D=64, ring=True)),
    (8, dict(B=1, S=8192, H=24, D=96, ring=True)),
    (4, dict(B=1, S=4096, H=8, D=128, stages=4, hostbuf=True)),   # host buffers in / out, pipelined per group
    (4, dict(B=1, S=3000, H=8, D=64, stages=2, n_src=3, hostbuf=True)),
    (4, dict(B=1, S=4096, H=8, D=128, usp=2)),                    # USP: Ulysses in pairs x Ring over 2 groups
    (8, dict(B=1, S=8192, H=12, D=64, usp=4)),
    # full size (configs[3]: 720p, 8 processes, N_st = 3), staged copy engines and direct stores
    (8, dict(B=1, S=118_800, H=24, D=128, stages=3, calls=2)),
    (8, dict(B=1, S=118_800, H=24, D=128, stages=3, calls=2, direct=True)),
])
def test_p2p_processes_bit_identical(world, case):
    _port_cache[0] = _port()
    _launch(world, case)
