#!/usr/bin/env python
"""Run torch SDPA (library kernels: cuDNN / flash) on one BASELINE-like shape a few times, for ncu to profile the
library's attention kernel next to ours (context only: prior art on the same hardware, not part of the product).

    ncu --set full -k regex:'^(?!.*(elementwise|fill|copy|memset)).*' -s 3 -c 1 python tools/sdpa_probe.py --shape hy76k
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

SHAPES = {"osp": (1, 28_800, 24, 96), "hy76k": (1, 76_032, 24, 128), "d64": (1, 32_768, 16, 64)}

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="hy76k")
ap.add_argument("--backend", default="cudnn")
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
B, S, H, D = SHAPES[a.shape]
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
be = {"cudnn": SDPBackend.CUDNN_ATTENTION, "flash": SDPBackend.FLASH_ATTENTION}[a.backend]
with sdpa_kernel(be):
    for _ in range(a.reps):
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
print("ok", a.shape, a.backend, float(o.float().abs().mean()))
