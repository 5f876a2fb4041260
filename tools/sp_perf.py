#!/usr/bin/env python
"""PipeSP on ONE GPU with P virtual ranks (loopback transport): whole-layer time per stage split,
with the library's per-step profile (attention, exchanges as device copies, pack/unpack).

The virtual ranks' work is serialised on one GPU, so this measures the per-stage overheads of the
schedule (kernel count, wave tails, copies), not multi-GPU speed.

    python tools/sp_perf.py [--workload hy720p129f] [--P 8] [--stages 1,3,24]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthgen  # noqa: E402
from paper_2511_12056_b200 import spa  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="hy720p129f")
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--stages", default="1,3,24")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--aco", type=int, default=0, help="n_src for an Aco plan (0 = PipeSP)")
    ap.add_argument("--ring", action="store_true", help="Ring-Attention plan instead of PipeSP")
    ap.add_argument("--pad", action="store_true", help="head padding when H % P != 0 (PAPER.md:196-199)")
    ap.add_argument("--direct", action="store_true", help="direct transport (SPA_OPT_DIRECT, loopback model of f1)")
    args = ap.parse_args()
    w = synthgen.WORKLOADS[args.workload]
    B, S, H, D, P = w.B, w.S, w.H, w.D, args.P
    nsrc = args.aco or P
    bnd = [0]
    for r in range(nsrc):   # uneven shards when nsrc does not divide S (first S % nsrc ranks one token longer)
        bnd.append(bnd[-1] + S // nsrc + (1 if r < S % nsrc else 0))
    shards = [[synthgen.gen_qkv_shard(0, t, (B, S, H, D), bnd[r], bnd[r + 1], device="cuda") for r in range(nsrc)]
              for t in range(3)]
    outs = [torch.empty_like(x) for x in shards[0]]
    flops = 4.0 * B * S * S * H * D
    q_all = torch.cat(shards[0], 1)
    k_all, v_all = torch.cat(shards[1], 1), torch.cat(shards[2], 1)
    o_all = torch.empty_like(q_all)
    for _ in range(2):
        spa.attention(q_all, k_all, v_all, o_all)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        spa.attention(q_all, k_all, v_all, o_all)
    b.record()
    torch.cuda.synchronize()
    t1 = a.elapsed_time(b) / args.reps
    print(json.dumps({"what": "single kernel, all heads", "ms": t1, "tflops": flops / t1 / 1e9}), flush=True)
    del q_all, k_all, v_all, o_all
    if args.ring:   # Ring-Attention plan (R21): P x P block attentions + merges, timed as a whole
        plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, ring=True)
        ws = plan.workspace()
        for _ in range(2):
            spa.spa_ring_attention_local(plan, *shards, outs, ws)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            spa.spa_ring_attention_local(plan, *shards, outs, ws)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.reps
        print(json.dumps({"ring": True, "P": P, "total_ms": ms, "tflops": flops / ms / 1e9}), flush=True)
        plan.close()
        return
    for st in [int(x) for x in args.stages.split(",")]:
        plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=st, n_src=args.aco, pad_heads=args.pad)
        if args.direct:
            plan.set_option(spa.SPA_OPT_DIRECT, 1)
        ws = plan.workspace()
        call = spa.spa_aco_attention_local if args.aco else spa.spa_pipesp_attention_local
        for _ in range(2):
            call(plan, *shards, outs, ws)
        torch.cuda.synchronize()
        plan.set_option(spa.SPA_OPT_PROFILE, 1)
        tot, att, ain, aout, pk, up = 0, 0, 0, 0, 0, 0
        for _ in range(args.reps):
            call(plan, *shards, outs, ws)
            torch.cuda.synchronize()
            pr = plan.last_profile()
            tot += pr.total_ms
            att += sum(pr.attn_ms[i] for i in range(pr.n_stages))
            ain += sum(pr.a2a_in_ms[i] for i in range(pr.n_stages))
            aout += sum(pr.a2a_out_ms[i] for i in range(pr.n_stages))
            pk += pr.pack_ms
            up += pr.unpack_ms
        r = args.reps
        print(json.dumps({"stages": st, "split": plan.stage_split, "P": P, "n_src": nsrc, "total_ms": tot / r,
                          "tflops": flops / (tot / r) / 1e9, "attn_ms_sum": att / r, "a2a_in_ms_sum": ain / r,
                          "a2a_out_ms_sum": aout / r, "pack_ms": pk / r, "unpack_ms": up / r,
                          "attn_launches": pr.attn_launches, "copy_launches": pr.copy_launches}), flush=True)
        plan.close()
        del ws


if __name__ == "__main__":
    main()
