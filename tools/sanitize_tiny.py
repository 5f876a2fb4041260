#!/usr/bin/env python
"""Tiny invocations of every library kernel for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_tiny.py [copy|merge|attn|qkv|all]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthgen  # noqa: E402
from paper_2511_12056_b200 import spa  # noqa: E402


def main(which):
    B, S, H, D, P = 1, 320, 4, 64, 2
    q, k, v = (synthgen.gen_qkv_shard(0, t, (B, S, H, D), 0, S, device="cuda") for t in range(3))
    S_l = S // P
    shards = [[x[:, r * S_l:(r + 1) * S_l].contiguous() for r in range(P)] for x in (q, k, v)]
    outs = [torch.empty_like(t) for t in shards[0]]
    if which in ("copy", "all"):   # pack / loopback exchange / unpack copy kernels (attention skipped: reshard)
        plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D)
        heads = [torch.empty((B, S, H // P, D), dtype=torch.bfloat16, device="cuda") for _ in range(P)]
        spa.spa_reshard_seq_to_head_local(plan, shards[0], heads, plan.workspace())
        spa.spa_reshard_head_to_seq_local(plan, heads, outs, plan.workspace())
        torch.cuda.synchronize()
        assert all(torch.equal(a, b) for a, b in zip(outs, shards[0]))
    if which in ("merge", "all"):  # ring: attention with fp32 partials + lse, then the lse merge kernel
        plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, ring=True)
        spa.spa_ring_attention_local(plan, *shards, outs, plan.workspace())
        torch.cuda.synchronize()
    if which in ("attn", "all"):
        spa.attention(q, k, v)
        plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=2)
        spa.spa_pipesp_attention_local(plan, *shards, outs, plan.workspace())
        torch.cuda.synchronize()
    if which in ("qkv", "all"):
        C = 128
        X = synthgen.gen_hidden_shard(0, (B, S, C), 0, S, device="cuda")
        plan = spa.Plan(spa.Comm.loopback(1), B, S, H, D)
        wp = plan.pack_qkv_weight(synthgen.gen_qkv_weight(0, C, H, D, device="cuda"),
                                  synthgen.gen_qkv_bias(0, H, D, device="cuda"))
        o = [torch.empty((B, S, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
        spa.spa_qkv_projection(plan, C, 0, X, wp, *o)
        torch.cuda.synchronize()
    print("sanitize_tiny ok:", which)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
