"""A real NCCL communicator on the one GPU available (nranks = 1): ncclCommInitRankConfig with an SM budget,
spa_comm_wait's completion / timeout / ncclCommAbort path, and an SP plan on the NCCL comm (SURVEY §5 failure
handling; the multi-rank NCCL exchange itself needs several GPUs -- see DESIGN.md §6)."""
import pytest
import torch

import synthgen
from paper_2511_12056_b200 import spa

pytestmark = pytest.mark.gpu


def test_nccl_config_plan_and_wait():
    comm = spa.Comm.nccl(spa.get_unique_id(), 1, 0, 0, min_ctas=1, max_ctas=4, cta_policy=1)
    B, S, H, D = 1, 2048, 4, 128
    q, k, v = (synthgen.gen_qkv_shard(0, t, (B, S, H, D), 0, S, device="cuda") for t in range(3))
    plan = spa.Plan(comm, B, S, H, D, stages=2)
    out = torch.empty_like(q)
    stream = torch.cuda.current_stream()
    spa.spa_pipesp_attention(plan, q, k, v, out, plan.workspace(), stream)
    comm.wait(stream, timeout_ms=60_000)
    assert torch.equal(out.view(torch.int16), spa.attention(q, k, v).view(torch.int16))
    comm.check()
    plan.close()
    comm.close()


def test_wait_timeout_aborts_the_communicator():
    comm = spa.Comm.nccl(spa.get_unique_id(), 1, 0, 0)
    w = synthgen.WORKLOADS["hy544p129f"]
    q, k, v = (synthgen.gen_qkv_shard(0, t, (w.B, w.S, w.H, w.D), 0, w.S, device="cuda") for t in range(3))
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    for _ in range(4):   # ~0.2 s of attention queued
        spa.attention(q, k, v, stream=stream)
    with pytest.raises(spa.SpaError) as e:
        comm.wait(stream, timeout_ms=1)
    assert e.value.status == 5 and "abort" in str(e.value)
    torch.cuda.synchronize()
    comm.close()


def test_nccl_symmetric_window_plumbing():
    """NCCL 2.28 symmetric windows (SURVEY f1 on NCCL plans): ncclMemAlloc + ncclCommWindowRegister, this rank's LSA
    address resolved with NCCL's device API, a kernel's stores through it visible at the local address."""
    comm = spa.Comm.nccl(spa.get_unique_id(), 1, 0, 0)
    comm.window_selftest(1 << 20)
    comm.window_selftest(64 << 20)
    with pytest.raises(spa.SpaError):
        comm.window_selftest(1000)   # not a multiple of 4096
    comm.close()


def test_nccl_window_plan_one_rank():
    """spa_plan_window_register on a 1-rank plan is a no-op; the window workspace serves the calls; ring plans and
    non-NCCL plans refuse the registration."""
    comm = spa.Comm.nccl(spa.get_unique_id(), 1, 0, 0)
    B, S, H, D = 1, 1024, 4, 64
    q, k, v = (synthgen.gen_qkv_shard(0, t, (B, S, H, D), 0, S, device="cuda") for t in range(3))
    plan = spa.Plan(comm, B, S, H, D, stages=2)
    ws = plan.window_setup()
    assert ws % 4096 == 0
    out = torch.empty_like(q)
    stream = torch.cuda.current_stream()
    spa.spa_pipesp_attention(plan, q, k, v, out, ws, stream)
    comm.wait(stream, timeout_ms=60_000)
    assert torch.equal(out.view(torch.int16), spa.attention(q, k, v).view(torch.int16))
    plan.close()
    ring = spa.Plan(comm, B, S, H, D, ring=True)
    with pytest.raises(spa.SpaError):
        ring.window_setup()
    ring.close()
    lb = spa.Plan(spa.Comm.loopback(2, 0), B, S, H, D)
    with pytest.raises(spa.SpaError):
        lb.window_setup()
    lb.close()
    comm.close()
