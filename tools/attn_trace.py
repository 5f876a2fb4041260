#!/usr/bin/env python
"""Per-iteration timeline of one attention CTA (debug build lib/libspa_trace.so, SPA_ATTN_TRACE).

    SPA_LIB=paper_2511_12056_b200/lib/libspa_trace.so python tools/attn_trace.py [--D 128]
Events (clock64 cycles) per KV iteration j of CTA (0,0,0):
  0/1  MMA issuer: P(j) key-half 0/1 ready (PV half issued)
  3/8  softmax key-half 0/1 (quarter-0 warp): before waiting for S(j)
  4/9  S(j) ready     5/10 row max exchanged     6/11 P half written and released
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthgen  # noqa: E402
from paper_2511_12056_b200 import spa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--D", type=int, default=128)
ap.add_argument("--S", type=int, default=32768)
ap.add_argument("--H", type=int, default=8)
args = ap.parse_args()
lib = spa.load()
q, k, v = (synthgen.gen_qkv_shard(0, t, (1, args.S, args.H, args.D), 0, args.S, device="cuda") for t in range(3))
for _ in range(2):
    spa.attention(q, k, v)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (256 * 16))()
lib.spa_debug_read_trace.argtypes = [ctypes.c_void_p]
assert lib.spa_debug_read_trace(ctypes.addressof(buf)) == 0
T = np.frombuffer(buf, dtype=np.uint64).reshape(256, 16).astype(np.int64)
t0 = T[0, 3]
n = min(256, (args.S + 127) // 128)
print("  j | mma: P0rdy   P1rdy | sm0: wait  Srdy   maxx   Pdone | sm1: wait  Srdy   maxx   Pdone")
for j in list(range(0, 8)) + list(range(n // 2, n // 2 + 4)) + list(range(n - 3, n)):
    r = T[j] - t0
    print(f"{j:3d} | {r[0]:8d} {r[1]:8d} | {r[3]:8d} {r[4]:8d} {r[5]:8d} {r[6]:8d} | {r[8]:8d} {r[9]:8d} {r[10]:8d} {r[11]:8d}"
          f" | qk: acq {r[12]:8d} got {r[13]:8d} | V: acq {r[14]:8d} got {r[15]:8d} | load K {r[2]:8d} V {r[7]:8d}")
mid = slice(n // 4, 3 * n // 4)
d = T[mid]
per = np.diff(d[:, 1]).mean()
ideal = {128: 1024, 96: 768, 64: 512}[args.D]
print(f"steady-state period per KV tile: {per:.0f} cycles (MMA-bound ideal {ideal} at D={args.D})")
# softmax events of tile j are written by the warps of tile parity j % 2 (base 3 or 8)
js = np.arange(n // 4, 3 * n // 4)
ev = np.stack([T[j, 3 + 5 * (j % 2): 7 + 5 * (j % 2)] for j in js])   # [tiles, 4]: loop top, S ready, max, P done
print(f"per tile (its parity's warps): wait S {np.mean(ev[:, 1] - ev[:, 0]):.0f}  max {np.mean(ev[:, 2] - ev[:, 1]):.0f}  "
      f"exp+store {np.mean(ev[:, 3] - ev[:, 2]):.0f}  (a parity handles every other tile)")
print(f"MMA: P(j) ready -> P(j+1) ready {np.mean(np.diff(T[js, 1])):.0f} cycles")
