"""C-ABI checks that need no GPU: the library loads, exports every symbol include/spa.h
declares, validates shapes synchronously, and its multi-rank host logic (pack jobs,
per-stage message lists, attention regions, Psi_g unpack) routes every element home."""
import ctypes

import numpy as np
import pytest

from paper_2511_12056_b200 import spa
from tests import hostsim

lib = spa.load()


def test_exports_every_header_symbol():
    names = spa.header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert b"sm_100a" in lib.spa_version()


def test_status_strings_and_pad_heads():
    assert lib.spa_status_string(0) == b"SPA_OK"
    assert lib.spa_status_string(6) == b"SPA_ERR_BUSY"
    assert spa.spa_pad_heads(24, 7) == (28, 4)
    assert spa.spa_pad_heads(8, 4) == (8, 0)
    assert spa.spa_pad_heads(5, 3) == (6, 1)


@pytest.mark.parametrize("shape,err", [
    (dict(B=1, S=256, H=4, D=80), 3),            # D unsupported
    (dict(B=1, S=1, H=4, D=64), 2),              # fewer tokens than ranks
    (dict(B=1, S=256, H=3, D=64), 2),            # H % P
    (dict(B=1, S=256, H=4, D=64, stages=0), 2),  # stages < 1
    (dict(B=1, S=4, H=2, D=64, stages=8), 2),    # more query chunks than local tokens
])
def test_plan_validation(shape, err):
    comm = spa.Comm.host(2, 0)
    with pytest.raises(spa.SpaError) as e:
        spa.Plan(comm, **shape)
    assert e.value.status == err


def test_pad_heads_flag_accepts_indivisible_heads():
    comm = spa.Comm.host(7, 0)
    with pytest.raises(spa.SpaError) as e:
        spa.Plan(comm, 1, 7 * 16, 24, 64)
    assert e.value.status == 2
    p = spa.Plan(comm, 1, 7 * 16, 24, 64, pad_heads=True)   # 24 heads on 7 GPUs -> 28
    assert p.stage_split == (1, 1, 4)
    # rank 6 owns padded heads 24..27 only: nothing to compute there
    assert spa.Plan(spa.Comm.host(7, 6), 1, 7 * 16, 24, 64, pad_heads=True).describe_attention(0, 6).n_heads == 0
    assert p.describe_attention(0, 5).n_heads == 4


@pytest.mark.parametrize("P,H,S,B,stages", [
    (4, 6, 32, 1, 1), (4, 6, 32, 2, 2), (3, 4, 36, 1, 2), (7, 24, 7 * 6, 1, 1), (7, 24, 7 * 6, 1, 4),
    (8, 20, 64, 1, 3), (2, 3, 16, 1, 2),
])
def test_host_path_padded_heads(P, H, S, B, stages):
    """Head padding: only real heads are packed, computed and unpacked."""
    D = 64
    plans = [spa.Plan(spa.Comm.host(P, r), B, S, H, D, stages=stages, pad_heads=True) for r in range(P)]
    xs, _ = _labels(B, S, H, D, P)
    outs = hostsim.run_path(plans, xs, xs, xs)
    for r in range(P):
        assert np.array_equal(outs[r], xs[r]), r
    Hp = -(-H // P) * P
    h = Hp // P
    G_h, C, g = plans[0].stage_split
    for r in range(P):
        for k in range(G_h * C):
            kh = k // C
            assert plans[r].describe_attention(k, r).n_heads == max(0, min(g, H - (r * h + kh * g)))


def test_ring_plan_validation_and_workspace():
    """Ring plans (R21): any H, S % P == 0; workspace = 2 K/V slots + P fp32 partials + lse."""
    P, B, S, H, D = 4, 2, 4 * 96, 5, 96
    p = spa.Plan(spa.Comm.host(P, 1), B, S, H, D, ring=True)
    E = B * (S // P) * H * D
    assert p.workspace_bytes >= 4 * E * 2 + P * E * 4 + P * (E // D) * 4
    with pytest.raises(spa.SpaError) as e:
        spa.Plan(spa.Comm.host(P, 0), B, S + 1, H, D, ring=True)
    assert e.value.status == 2
    with pytest.raises(spa.SpaError) as e:   # Ulysses / PipeSP calls refuse a ring plan before anything else
        spa.spa_pipesp_attention(p, 16, 16, 16, 16, 16, stream=0)
    assert e.value.status == 1
    with pytest.raises(spa.SpaError):
        p.describe_messages(0, 0, 1)
    assert spa.Plan(spa.Comm.host(1, 0), B, S, H, D, ring=True).workspace_bytes == 0
    for kw in (dict(stages=2), dict(pad_heads=True), dict(stages=3, ulysses=2)):   # spa.h: stages 1, pad_heads 0
        with pytest.raises(spa.SpaError) as e:
            spa.Plan(spa.Comm.host(P, 0), B, S, 4, D, ring=True, **kw)
        assert e.value.status == 1, kw


def test_usp_plan_validation():
    """USP hybrid: Ulysses degree U | nranks and U | H; sub-plans on sub-comms."""
    p = spa.Plan(spa.Comm.host(8, 3), 1, 8 * 64, 12, 128, ring=True, ulysses=4)
    assert p.workspace_bytes > 4 * 64 * 12 * 128 * 2
    for kw, err in [(dict(ulysses=3), 2), (dict(ulysses=8, H=12), 2)]:
        H = kw.pop("H", 12)
        with pytest.raises(spa.SpaError) as e:
            spa.Plan(spa.Comm.host(8, 0), 1, 8 * 64, H, 128, ring=True, **kw)
        assert e.value.status == err
    with pytest.raises(spa.SpaError) as e:
        spa.Plan(spa.Comm.host(8, 0), 1, 8 * 64, 12, 128, ulysses=4)   # needs ring = 1
    assert e.value.status == 1


def test_host_comm_cannot_execute():
    comm = spa.Comm.host(2, 1)
    plan = spa.Plan(comm, 1, 256, 4, 64, stages=2)
    with pytest.raises(spa.SpaError) as e:
        spa.spa_pipesp_attention(plan, 16, 16, 16, 16, 16, stream=0)
    assert e.value.status == 3


def test_stage_split_and_workspace():
    comm = spa.Comm.host(8, 0)
    for st, exp in [(1, (1, 1, 3)), (3, (3, 1, 1)), (4, (1, 4, 3)), (24, (3, 8, 1)), (6, (3, 2, 1))]:
        p = spa.Plan(comm, 1, 118_800, 24, 128, stages=st)
        assert p.stage_split == exp
        shard = 118_800 // 8 * 24 * 128 * 2
        # 8 exchange shards + the direct transport's landing shard + the epoch-flag block (P2P / NCCL-window plans;
        # DESIGN.md §4)
        flags = 4 * 8 * (1 + 2 * exp[0] * exp[1])
        assert shard * 9 + flags <= p.workspace_bytes < shard * 9 + flags + 10 * 256


def _labels(B, S, H, D, P, n_src=None):
    """per-source label shards (uneven when n_src does not divide S: the first S % n_src ranks get one more)"""
    n_src = n_src or P
    bnd = [0]
    for r in range(n_src):
        bnd.append(bnd[-1] + S // n_src + (1 if r < S % n_src else 0))
    b = np.arange(B)[:, None, None, None]
    s = np.arange(S)[None, :, None, None]
    k = np.arange(H)[None, None, :, None]
    d = np.arange(D)[None, None, None, :]
    X = ((b * 7 + s * 131 + k * 17 + d) % 65521).astype(np.uint16)
    return [np.ascontiguousarray(X[:, bnd[r]:bnd[r + 1]]).view(np.uint8).reshape(-1) for r in range(n_src)], X


@pytest.mark.parametrize("P,H,S,B,stages", [
    (2, 4, 32, 1, 1), (2, 4, 32, 1, 2), (2, 4, 32, 2, 4), (4, 8, 64, 1, 2), (4, 8, 64, 1, 6),
    (8, 24, 96, 1, 1), (8, 24, 96, 1, 3), (8, 24, 96, 1, 4), (8, 24, 96, 1, 24), (3, 6, 36, 2, 4),
])
def test_host_path_routes_every_element_home(P, H, S, B, stages):
    D = 64
    plans = [spa.Plan(spa.Comm.host(P, r), B, S, H, D, stages=stages) for r in range(P)]
    xs, _ = _labels(B, S, H, D, P)
    outs = hostsim.run_path(plans, xs, xs, xs)
    for r in range(P):
        assert np.array_equal(outs[r], xs[r]), r


@pytest.mark.parametrize("P,H,S,B,stages", [
    (3, 6, 29, 1, 1), (3, 6, 29, 2, 2), (7, 7, 7 * 5 + 3, 1, 1), (4, 8, 4 * 6 + 3, 1, 4), (8, 24, 8 * 11 + 7, 1, 24),
    (2, 4, 9, 1, 2),
])
def test_host_path_uneven_shards(P, H, S, B, stages):
    """S % P != 0 (R9): shards differ by one token; every element still routes home."""
    D = 64
    plans = [spa.Plan(spa.Comm.host(P, r), B, S, H, D, stages=stages) for r in range(P)]
    xs, _ = _labels(B, S, H, D, P)
    outs = hostsim.run_path(plans, xs, xs, xs)
    for r in range(P):
        assert np.array_equal(outs[r], xs[r]), r


@pytest.mark.parametrize("n_src,N,H,S,stages", [(7, 8, 24, 7 * 12 + 3, 1), (7, 8, 24, 7 * 12 + 5, 3)])
def test_host_path_aco_seven_plus_one(n_src, N, H, S, stages):
    """The paper's Aco example: 24 heads, 7 denoising GPUs + 1 decoding GPU -- owners hold 3
    heads each, the sequence is sharded over 7 (unevenly)."""
    B, D = 1, 64
    plans = [spa.Plan(spa.Comm.host(N, r), B, S, H, D, stages=stages, n_src=n_src) for r in range(N)]
    xs, _ = _labels(B, S, H, D, N, n_src)
    outs = hostsim.run_path(plans, xs, xs, xs)
    for r in range(n_src):
        assert np.array_equal(outs[r], xs[r])


@pytest.mark.parametrize("n_src,N,H,stages", [(6, 8, 24, 1), (6, 8, 24, 3), (3, 4, 8, 2), (1, 2, 2, 1)])
def test_host_path_aco(n_src, N, H, stages):
    B, S, D = 1, 12 * n_src, 64
    plans = [spa.Plan(spa.Comm.host(N, r), B, S, H, D, stages=stages, n_src=n_src) for r in range(N)]
    xs, _ = _labels(B, S, H, D, N, n_src)
    outs = hostsim.run_path(plans, xs, xs, xs)
    for r in range(n_src):
        assert np.array_equal(outs[r], xs[r])
    # co-processors send nothing on the input side and receive nothing on the output side
    for r in range(n_src, N):
        assert not plans[r].describe_pack(r) and not plans[r].describe_unpack(r)
        assert all(m.is_recv for m in plans[r].describe_messages(0, 0, r))
        assert not any(m.is_recv for m in plans[r].describe_messages(0, 1, r))


def test_messages_stay_inside_workspace():
    P = 4
    plans = [spa.Plan(spa.Comm.host(P, r), 2, 64, 8, 96, stages=4) for r in range(P)]
    nb = plans[0].workspace_bytes
    for r in range(P):
        for k in range(4):
            for d in (0, 1):
                for m in plans[r].describe_messages(k, d, r):
                    assert 0 <= m.off and m.off + m.bytes <= nb and m.off % 16 == 0 and m.bytes % 64 == 0
            a = plans[r].describe_attention(k, r)
            assert a.q_off % 16 == 0 and a.o_off % 16 == 0 and a.Skv == 64


def test_plain_c_client(tmp_path):
    """The boundary is a C ABI: a plain C program (tests/c_abi/abi_smoke.c) compiled with gcc against
    include/spa.h and libspa.so creates plans and reads their descriptions without Python or torch."""
    import os
    import subprocess
    from paper_2511_12056_b200 import _build
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = _build.build()
    exe = str(tmp_path / "abi_smoke")
    subprocess.check_call(["gcc", "-std=c11", "-O1", "-I", os.path.join(root, "include"),
                           os.path.join(root, "tests", "c_abi", "abi_smoke.c"), lib, "-o", exe,
                           f"-Wl,-rpath,{os.path.dirname(lib)}"])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    assert "c abi ok" in out.stdout


def test_p2p_comm_needs_a_device():
    """spa_comm_init_p2p (CUDA IPC transport) fails cleanly without a GPU: SPA_ERR_CUDA, nothing created."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by tests/test_gpu_p2p.py")
    with pytest.raises(spa.SpaError) as e:
        spa.Comm.p2p(2, 0, 0)
    assert e.value.status == 4


@pytest.mark.parametrize("cfg", [dict(min_ctas=-1), dict(min_ctas=8, max_ctas=4), dict(cta_policy=3)])
def test_nccl_config_validated_before_any_call(cfg):
    """spa_comm_init_config rejects bad NCCL SM budgets synchronously (SPA_ERR_INVALID), before touching CUDA/NCCL."""
    with pytest.raises(spa.SpaError) as e:
        spa.Comm.nccl(b"\0" * 128, 2, 0, 0, **{"min_ctas": 0, "max_ctas": 0, "cta_policy": 0, **cfg})
    assert e.value.status == 1


def _match(msgs_of, P):
    """For every ordered pair (p, q): p's sends to q and q's receives from p, in issue order, pair up one to one
    with equal sizes (NCCL's matching rule) -- returns the pairs."""
    pairs = []
    for p in range(P):
        for q in range(P):
            sends = [m for m in msgs_of[p] if not m.is_recv and m.peer == q]
            recvs = [m for m in msgs_of[q] if m.is_recv and m.peer == p]
            assert len(sends) == len(recvs), (p, q)
            for s, r in zip(sends, recvs):
                assert s.bytes == r.bytes
                pairs.append((p, s, q, r))
    return pairs


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_ring_messages_match_and_rotate(P):
    """Ring plans (R21): every step's sends and receives match across ranks, and after step t rank r's receive slot
    t&1 holds the K/V block of rank (r - t - 1) mod P (simulated on block labels)."""
    B, S, H, D = 1, P * 32, 3, 64
    plans = [spa.Plan(spa.Comm.host(P, r), B, S, H, D, ring=True) for r in range(P)]
    held = {r: {("K", None): r, ("V", None): r} for r in range(P)}   # block label per (buffer, ws offset)
    for t in range(P - 1):
        msgs = {r: plans[r].describe_ring(t, r) for r in range(P)}
        new = {r: dict(held[r]) for r in range(P)}
        for p, s, q, r in _match(msgs, P):
            key = ("K", None) if s.buf == spa.BUF_K else ("V", None) if s.buf == spa.BUF_V else ("WS", s.off)
            new[q][("WS", r.off)] = held[p][key]
        held = new
        for r in range(P):
            k_slot, v_slot = [m.off for m in msgs[r] if m.is_recv]
            assert held[r][("WS", k_slot)] == held[r][("WS", v_slot)] == (r - t - 1) % P


@pytest.mark.parametrize("P,U", [(4, 2), (8, 2), (8, 4)])
def test_usp_messages_match(P, U):
    """USP (R21): the ring steps of every Ulysses index u match across the R = P/U ranks of that ring (global peers),
    and the Ulysses group exchange (a seq->head reshard over U ranks) matches inside every group."""
    B, S, H, D = 1, P * 16, 4 * U, 64
    plans = [spa.Plan(spa.Comm.host(P, r), B, S, H, D, ring=True, ulysses=U) for r in range(P)]
    R = P // U
    for t in range(max(1, R - 1)):
        msgs = {r: plans[r].describe_ring(t, r) for r in range(P)}
        for p, s, q, r in _match(msgs, P):
            assert p % U == q % U and q == ((p // U + 1) % R) * U + p % U
    sub = [spa.Plan(spa.Comm.host(U, u), B, U * (S // P), H, D) for u in range(U)]
    for d in (0, 1):
        _match({u: sub[u].describe_messages(0, d, u) for u in range(U)}, U)


def test_window_register_needs_an_nccl_plan():
    """spa_plan_window_register (NCCL symmetric windows) refuses host plans and NULL arguments before
    touching any device; the direct option is accepted at set-up on NCCL-like plans and checked at the call."""
    lib = spa.load()
    p = spa.Plan(spa.Comm.host(4, 1), 1, 64, 8, 64, stages=2)
    assert lib.spa_plan_window_register(p.h, ctypes.c_void_p(4096)) == 1   # SPA_ERR_INVALID: not an NCCL plan
    assert b"NCCL" in lib.spa_last_error()
    assert lib.spa_plan_window_register(p.h, None) == 1
    assert lib.spa_mem_free(None) == 0
    p.set_option(spa.SPA_OPT_DIRECT, 1)
    p.close()
