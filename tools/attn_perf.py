#!/usr/bin/env python
"""Attention-kernel sweep (CUDA events, L2 flushed between reps): ms and TFLOP/s per shape.
Context comparison: torch SDPA (cuDNN / flash backend) on the same inputs (not a target).

    python tools/attn_perf.py [--reps 10] [--sdpa] [--shapes osp,hy76k,hy720p8,d64]
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

SHAPES = {
    "osp": (1, 28_800, 24, 96),
    "hy76k": (1, 76_032, 24, 128),
    "hy720p8": (1, 118_800, 3, 128),   # one rank's heads at P=8 (full sequence)
    "d64": (1, 32_768, 16, 64),
    "osp_p8": (1, 28_800, 3, 96),
}


def bench(fn, reps, flush):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--sdpa", action="store_true")
    ap.add_argument("--shapes", default=",".join(SHAPES))
    args = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in args.shapes.split(","):
        B, S, H, D = SHAPES[name]
        q, k, v = (synthgen.gen_qkv_shard(0, t, (B, S, H, D), 0, S, device="cuda") for t in range(3))
        out = torch.empty_like(q)
        flops = 4.0 * B * S * S * H * D
        ms = bench(lambda: spa.attention(q, k, v, out), args.reps, flush)
        rec = {"shape": name, "B": B, "S": S, "H": H, "D": D, "ms": ms, "tflops": flops / ms / 1e9}
        if args.sdpa:
            qt, kt, vt = (x.transpose(1, 2).contiguous() for x in (q, k, v))
            try:
                ms2 = bench(lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt), args.reps, flush)
                rec["torch_sdpa_ms"] = ms2
                rec["torch_sdpa_tflops"] = flops / ms2 / 1e9
            except Exception as e:  # pragma: no cover
                rec["torch_sdpa_error"] = str(e)[:200]
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
