#!/usr/bin/env python
"""Throughput of the QKV-projection GEMM (qkv_gemm.cu) on one GPU, CUDA events, L2 flushed:
the whole-sequence projection of a 1-rank plan (M = B*S tokens) and one rank's projections at P = 8 (M = S/8, one
GEMM per head group), against the measured bf16 peak; torch.matmul (cuBLAS) on the same shapes as context.

    python tools/qkv_perf.py [--workloads hy544p129f,hy720p129f] [--reps 10]
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


def timed(fn, reps, flush):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="osp480p93f,hy544p129f,hy720p129f")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1652.2
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in args.workloads.split(","):
        w = synthgen.WORKLOADS[name]
        B, S, H, D = w.B, w.S, w.H, w.D
        C = H * D
        W = synthgen.gen_qkv_weight(0, C, H, D, device="cuda")
        bias = synthgen.gen_qkv_bias(0, H, D, device="cuda")
        for P, stages in ((1, 1), (8, 3)):
            S_r = S // P
            X = synthgen.gen_hidden_shard(0, (B, S, C), 0, S_r, device="cuda")
            plan = spa.Plan(spa.Comm.loopback(P), B, S, H, D, stages=stages)
            wp = plan.pack_qkv_weight(W, bias)
            q, k, v = (torch.empty((B, S_r, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(3))
            ms = timed(lambda: spa.spa_qkv_projection(plan, C, 0, X, wp, q, k, v), args.reps, flush)
            flops = 2.0 * B * S_r * C * 3 * H * D
            Wt = W.t().contiguous()
            ms_cublas = timed(lambda: torch.matmul(X.view(-1, C), W.t()), args.reps, flush)
            print(json.dumps({"workload": name, "P": P, "M": B * S_r, "N": 3 * H * D, "K": C,
                              "head_groups": plan.stage_split[0], "ms": ms, "tflops": flops / ms / 1e9,
                              "frac_of_peak": flops / ms / 1e9 / peak, "cublas_ms": ms_cublas,
                              "cublas_tflops": flops / ms_cublas / 1e9}), flush=True)
            plan.close()
            del X, q, k, v, wp, Wt


if __name__ == "__main__":
    main()
