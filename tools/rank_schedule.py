#!/usr/bin/env python
"""One rank's share of the P-GPU PipeSP schedule, MEASURED on one GPU (SPA_OPT_RANK_ONLY): a loopback plan over P
virtual ranks runs only virtual rank r's launches -- its pack (or fused QKV projection), its attention stages, its
unpack -- and only the messages rank r sends or receives, through the library's real scheduler (comm stream, events,
alternating compute streams).  What this captures that a single-launch time does not: per-stage wave tails, the
stage-to-stage overlap, and the SM contention between the exchange copies and the attention grid.

Transports: `kernel` = the copy kernel moves the bytes on SMs (as NCCL's kernels would), `ce` = copy-engine
cudaMemcpyAsync (the P2P transport's staged exchange, no SMs), `direct` = pack and attention epilogue store to the
owners themselves (SPA_OPT_DIRECT), `skip` = no exchange (the exposed-communication baseline).  Local copies move
bytes at HBM speed; the line also carries the bytes this rank puts on NVLink and their time at 900 GB/s.

    python tools/rank_schedule.py [--workloads hy720p129f,osp480p93f] [--P 8] [--stages 1,2,3,4,6,8,12,24]
                                  [--modes skip,kernel,ce,direct] [--qkv]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthgen  # noqa: E402
from paper_2511_12056_b200 import spa  # noqa: E402


def sent_bytes(plan, rank):
    n = 0
    G_h, C, _ = plan.stage_split
    for k in range(G_h * C):
        for d in (0, 1):
            n += sum(m.bytes for m in plan.describe_messages(k, d, rank) if not m.is_recv and m.peer != rank)
    return n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="hy720p129f,osp480p93f")
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--stages", default="1,2,3,4,6,8,12,24")
    ap.add_argument("--modes", default="skip,kernel,ce,direct")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--qkv", action="store_true", help="layer from hidden states (fused QKV projection, f3)")
    ap.add_argument("--window", type=int, default=4, help="SPA_OPT_STAGE_WINDOW (stages in flight)")
    ap.add_argument("--aco", type=int, default=0,
                    help="Aco plan: n_src source ranks of P (PAPER.md:150-199); --rank may name a co-processor")
    ap.add_argument("--peak", type=float, default=None, help="bf16 TF/s (default MEASURED_PEAKS.json)")
    args = ap.parse_args()
    peak = args.peak
    if peak is None:
        try:
            peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
        except Exception:
            peak = 1652.2
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    P, r = args.P, args.rank
    for name in args.workloads.split(","):
        w = synthgen.WORKLOADS[name]
        B, S, H, D = w.B, w.S, w.H, w.D
        nsrc = args.aco or P
        bnd = [0]   # source shards differ by <= 1 token (R9)
        for q in range(nsrc):
            bnd.append(bnd[-1] + S // nsrc + (1 if q < S % nsrc else 0))
        S_l = S // nsrc
        C = H * D
        if args.qkv:
            xs = [synthgen.gen_hidden_shard(0, (B, S, C), bnd[q], bnd[q + 1], device="cuda") for q in range(P)]
            W = synthgen.gen_qkv_weight(0, C, H, D, device="cuda")
            bias = synthgen.gen_qkv_bias(0, H, D, device="cuda")
        else:
            shards = [[synthgen.gen_qkv_shard(0, t, (B, S, H, D), bnd[q], bnd[q + 1], device="cuda")
                       for q in range(nsrc)] for t in range(3)]
        outs = [torch.empty((B, bnd[q + 1] - bnd[q], H, D), dtype=torch.bfloat16, device="cuda") for q in range(nsrc)]
        attn_flops_rank = 4.0 * B * S * S * H * D / P
        proj_flops_rank = 2.0 * B * S_l * C * 3 * H * D if args.qkv else 0.0
        if args.qkv and args.aco:
            raise SystemExit("--qkv plans have no co-processor ranks")
        for st in [int(x) for x in args.stages.split(",")]:
            plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=st, n_src=args.aco)
            plan.set_option(spa.SPA_OPT_STAGE_WINDOW, args.window)
            ws = plan.qkv_workspace() if args.qkv else plan.workspace()
            wp = plan.pack_qkv_weight(W, bias) if args.qkv else None
            nbytes = sent_bytes(plan, r)
            # one full call (all virtual ranks) first: every buffer the rank-only calls read then holds real data --
            # the attention's power draw, and so the power-capped clock, depends on the operand values
            plan.set_option(spa.SPA_OPT_RANK_ONLY, 0)
            sp_call = spa.spa_aco_attention_local if args.aco else spa.spa_pipesp_attention_local
            if args.qkv:
                spa.spa_pipesp_qkv_attention_local(plan, C, xs, wp, outs, ws)
            else:
                sp_call(plan, *shards, outs, ws)
            torch.cuda.synchronize()
            res = {}
            for mode in args.modes.split(","):
                plan.set_option(spa.SPA_OPT_RANK_ONLY, r + 1)
                plan.set_option(spa.SPA_OPT_LOOPBACK_CE, int(mode == "ce"))
                plan.set_option(spa.SPA_OPT_DIRECT, int(mode == "direct"))
                plan.set_option(spa.SPA_OPT_SKIP_COMM, int(mode == "skip"))

                def call():
                    if args.qkv:
                        spa.spa_pipesp_qkv_attention_local(plan, C, xs, wp, outs, ws)
                    else:
                        sp_call(plan, *shards, outs, ws)
                for _ in range(2):
                    call()
                torch.cuda.synchronize()
                ts, prof = [], []
                plan.set_option(spa.SPA_OPT_PROFILE, 1)
                for _ in range(args.reps):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    call()
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                    prof.append(plan.last_profile())
                plan.set_option(spa.SPA_OPT_PROFILE, 0)
                ms = statistics.median(ts)
                pm = prof[len(prof) // 2]
                res[mode] = ms
                t_roof = max((attn_flops_rank + proj_flops_rank) / (peak * 1e12), nbytes / 900e9) * 1e3
                rec = {"workload": name, "P": P, "n_src": nsrc, "rank": r, "stages": st, "window": args.window, "stage_split": list(plan.stage_split),
                       "mode": mode, "qkv": args.qkv, "ms_per_layer": ms,
                       "tflops_per_gpu": (attn_flops_rank + proj_flops_rank) / (ms * 1e-3) / 1e12,
                       "tflops_aggregate_if_P_gpus": P * (attn_flops_rank + proj_flops_rank) / (ms * 1e-3) / 1e12,
                       "frac_overlapped_roofline": t_roof / ms, "t_roofline_ms": t_roof,
                       "attn_ms_sum": sum(pm.attn_ms[k] for k in range(pm.n_stages)),
                       "pack_ms": pm.pack_ms, "unpack_ms": pm.unpack_ms,
                       "a2a_in_ms_sum": sum(pm.a2a_in_ms[k] for k in range(pm.n_stages)),
                       "a2a_out_ms_sum": sum(pm.a2a_out_ms[k] for k in range(pm.n_stages)),
                       "nvlink_bytes_sent": nbytes, "nvlink_ms_at_900": nbytes / 900e9 * 1e3,
                       "launches": pm.attn_launches + pm.copy_launches + pm.gemm_launches}
                if "skip" in res and mode != "skip":
                    rec["exposed_pct_vs_skip"] = max(0.0, (ms - res["skip"]) / ms * 100)
                print(json.dumps(rec), flush=True)
            plan.close()
            del ws, wp


if __name__ == "__main__":
    main()
