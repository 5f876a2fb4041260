#!/usr/bin/env python
"""Interleaved A/B timing of attention-kernel builds in ONE process (tools/variants.py builds them).

Every round times each variant once per shape (L2 flushed before each launch, CUDA events), cycling the
variants in a rotating order, so power-cap / thermal drift on the box hits all variants alike.  Prints, per
(shape, variant), the median TF/s and the median of the per-round ratio to the first variant.

    python tools/ab.py base lea ... [--shapes osp,hy76k,d64] [--rounds 15]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthgen  # noqa: E402

SHAPES = {
    "osp": (1, 28_800, 24, 96),
    "hy76k": (1, 76_032, 24, 128),
    "hy720p8": (1, 118_800, 3, 128),
    "d64": (1, 32_768, 16, 64),
    "osp_p8": (1, 28_800, 3, 96),
    "hy544p8": (1, 76_032, 3, 128),
}


def lib_path(name):
    d = os.path.join(ROOT, "paper_2511_12056_b200", "lib")
    return os.path.join(d, "libspa.so" if name == "base" else f"libspa_{name}.so")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="+")
    ap.add_argument("--shapes", default="osp,hy76k,d64")
    ap.add_argument("--rounds", type=int, default=15)
    args = ap.parse_args()
    P, LL = ctypes.c_void_p, ctypes.c_longlong
    libs = []
    for v in args.variants:
        lib = ctypes.CDLL(lib_path(v), mode=ctypes.RTLD_LOCAL)
        f = lib.spa_attention_fwd
        f.argtypes = [P, P, P, P] + [ctypes.c_int] * 5 + [LL] * 6 + [P]
        f.restype = ctypes.c_int
        libs.append(f)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for shape in args.shapes.split(","):
        B, S, H, D = SHAPES[shape]
        q, k, v = (synthgen.gen_qkv_shard(0, t, (B, S, H, D), 0, S, device="cuda") for t in range(3))
        out = torch.empty_like(q)
        flops = 4.0 * B * S * S * H * D
        st = torch.cuda.current_stream().cuda_stream

        def call(f):
            r = f(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), B, S, S, H, D, H * D, S * H * D, H * D,
                  S * H * D, H * D, S * H * D, st)
            assert r == 0, r

        for f in libs:   # warm up every variant
            for _ in range(2):
                call(f)
        torch.cuda.synchronize()
        ts = [[] for _ in libs]
        n = len(libs)
        for rnd in range(args.rounds):
            for i in range(n):
                j = (i + rnd) % n
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                call(libs[j])
                b.record()
                torch.cuda.synchronize()
                ts[j].append(a.elapsed_time(b))
        med = [sorted(t)[len(t) // 2] for t in ts]
        for j, name in enumerate(args.variants):
            ratios = sorted(ts[0][r] / ts[j][r] for r in range(args.rounds))
            print(json.dumps({"shape": shape, "variant": name, "ms": med[j], "tflops": flops / med[j] / 1e9,
                              "speedup_vs_first": ratios[len(ratios) // 2], "S": S, "H": H, "D": D,
                              "rounds": args.rounds}), flush=True)


if __name__ == "__main__":
    main()
