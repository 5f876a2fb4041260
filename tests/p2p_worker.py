"""Worker of the multi-process P2P tests (tests/test_gpu_p2p.py): one process per rank, all on cuda:0.

Each rank generates only its own sequence shard (synthgen), sets up the P2P plan over CUDA IPC (handles exchanged
through a gloo process group), runs the SP call several times, and compares its output shard bit for bit with the
single-GPU kernel on the full (regenerated) inputs -- the same bits every path must produce (R18)."""
from __future__ import annotations

import os
import traceback


def run(rank: int, world: int, port: int, case: dict, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist

        import synthgen
        from paper_2511_12056_b200 import spa
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        B, S, H, D = case["B"], case["S"], case["H"], case["D"]
        n_src = case.get("n_src", 0) or world
        bounds = [0]
        for r in range(n_src):
            bounds.append(bounds[-1] + S // n_src + (1 if r < S % n_src else 0))
        src = rank < n_src
        usp = case.get("usp", 0)   # Ulysses degree of a USP plan (ring over the groups)
        ring = case.get("ring", False) or usp > 1
        plan = spa.Plan(spa.Comm.p2p(world, rank, 0), B, S, H, D, stages=case.get("stages", 1),
                        n_src=case.get("n_src", 0), ring=ring, ulysses=usp)
        if case.get("direct"):
            plan.set_option(spa.SPA_OPT_DIRECT, 1)
        ws = torch.empty(plan.host_sp_workspace_bytes, dtype=torch.uint8, device="cuda") if case.get("hostbuf") \
            else plan.workspace()
        plan.ipc_setup(ws)
        qkv_mode = case.get("qkv", False)
        if qkv_mode:
            C = H * D
            X = synthgen.gen_hidden_shard(1, (B, S, C), 0, S, device="cuda")
            W = synthgen.gen_qkv_weight(1, C, H, D, device="cuda")
            bias = synthgen.gen_qkv_bias(1, H, D, device="cuda")
            wp = plan.pack_qkv_weight(W, bias)
            x_r = X[:, bounds[rank]:bounds[rank + 1]].contiguous()
            p1 = spa.Plan(spa.Comm.loopback(1), B, S, H, D)
            full = [torch.empty((B, S, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
            spa.spa_qkv_projection(p1, C, 0, X, p1.pack_qkv_weight(W, bias), *full)
        else:
            full = [synthgen.gen_qkv_shard(case.get("seed", 0), t, (B, S, H, D), 0, S, device="cuda")
                    for t in range(3)]
        if ring:   # the ring's reference bits: the same plan over `world` virtual ranks on one GPU (R21)
            lp = spa.Plan(spa.Comm.loopback(world), B, S, H, D, ring=True, ulysses=usp)
            parts = [[x[:, bounds[r]:bounds[r + 1]].contiguous() for r in range(world)] for x in full]
            louts = [torch.empty_like(t) for t in parts[0]]
            spa.spa_ring_attention_local(lp, *parts, louts, lp.workspace())
            ref = torch.cat(louts, dim=1)
        else:
            ref = spa.attention(*full)
        torch.cuda.synchronize()
        out = torch.empty((B, bounds[rank + 1] - bounds[rank], H, D), dtype=torch.bfloat16, device="cuda") \
            if src else None
        shard = [x[:, bounds[rank]:bounds[rank + 1]].contiguous() for x in full] if src else [None] * 3
        for it in range(case.get("calls", 3)):
            if out is not None:
                out.fill_(0)
            if case.get("hostbuf"):   # pinned host buffers in and out (spa_pipesp_attention_hostbuf)
                hq = [x.cpu().pin_memory() if x is not None else None for x in shard]
                hout = torch.zeros(out.shape, dtype=out.dtype).pin_memory() if src else None
                spa.spa_pipesp_attention_hostbuf(plan, *hq, hout, ws)
                torch.cuda.synchronize()
                if src:
                    out.copy_(hout)
            elif qkv_mode:
                spa.spa_pipesp_qkv_attention(plan, C, x_r, wp, out, ws)
            elif ring:
                spa.spa_ring_attention(plan, *shard, out, ws)
            elif case.get("n_src"):
                spa.spa_aco_attention(plan, *shard, out, ws)
            elif case.get("ulysses"):
                spa.spa_ulysses_attention(plan, *shard, out, ws)
            else:
                spa.spa_pipesp_attention(plan, *shard, out, ws)
            torch.cuda.synchronize()
            if src:
                exp = ref[:, bounds[rank]:bounds[rank + 1]]
                if not torch.equal(out.view(torch.int16), exp.view(torch.int16)):
                    bad = (out.float() - exp.float()).abs().max().item()
                    raise AssertionError(f"rank {rank} call {it}: output differs from the single-GPU kernel "
                                         f"(max diff {bad})")
        dist.barrier()
        plan.close()
        dist.destroy_process_group()
    except Exception:
        errq.put((rank, traceback.format_exc()))
        raise
