#!/usr/bin/env python
"""Per-rank attention time of SP at P = 1, 2, 4, 8 measured on ONE GPU: the kernel on one rank's heads
(H/P heads over the full sequence, exactly the launch a rank makes with N_st = 1) for the BASELINE
workloads, CUDA events, L2 flushed.  With the all-to-all volume per rank and the NVLink 5 bandwidth this
gives the projected per-layer time of DESIGN.md (a model: the multi-GPU run itself needs N GPUs).

    python tools/per_rank_perf.py [--reps 5]
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
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nvlink-gbs", type=float, default=900.0)
    ap.add_argument("--hbm-gbs", type=float, default=6553.6)
    args = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in ("osp480p93f", "hy544p129f", "hy720p129f"):
        w = synthgen.WORKLOADS[name]
        for P in (1, 2, 4, 8):
            h = w.H // P
            q, k, v = (synthgen.gen_qkv_shard(0, t, (w.B, w.S, h, w.D), 0, w.S, device="cuda") for t in range(3))
            out = torch.empty_like(q)
            for _ in range(2):
                spa.attention(q, k, v, out)
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                spa.attention(q, k, v, out)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            ms = ts[len(ts) // 2]
            flops = 4.0 * w.B * w.S * w.S * h * w.D
            shard = w.B * (w.S // P) * w.H * w.D * 2
            a2a_ms = (4 * shard * (P - 1) / P) / (args.nvlink_gbs * 1e9) * 1e3   # Q, K, V in + O out
            copy_ms = (2 * 4 * shard) / (args.hbm_gbs * 1e9) * 1e3 if P > 1 else 0.0   # pack + unpack
            print(json.dumps({"workload": name, "P": P, "heads_per_rank": h, "attn_ms": ms,
                              "tflops_per_gpu": flops / ms / 1e9, "a2a_ms_model": a2a_ms,
                              "pack_unpack_ms_model": copy_ms,
                              "layer_ms_if_overlapped": ms + copy_ms + (a2a_ms / h if P > 1 else 0.0)}),
                  flush=True)
            del q, k, v, out


if __name__ == "__main__":
    main()
