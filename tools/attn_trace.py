#!/usr/bin/env python
"""Per-iteration timeline of one attention CTA (debug build lib/libspa_trace.so, SPA_ATTN_TRACE).

    SPA_LIB=paper_2511_12056_b200/lib/libspa_trace.so python tools/attn_trace.py [--D 128]
Events (clock64 cycles) per KV iteration j of CTA (0,0,0):
  0 MMA: before waiting P0(j)   1 MMA: P0(j) ready (PV0 issue)   2 MMA: P1(j) ready (PV1 issue)
  3/8 softmax t0/t1: before S wait   4/9 S ready   5/10 S in registers   6/11 exps done   7/12 P signalled
  14/15 producer: K_j / V_j slot free
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
print("j  | mma0:kv-ok P0a-rdy  mma1:P1a-rdy | s0: wait  rdy  ld  exp  sig | s1: wait rdy  ld  exp  sig | kfree vfree")
for j in list(range(0, 12)) + list(range(n // 2, n // 2 + 6)) + list(range(n - 4, n)):
    r = T[j] - t0
    print(f"{j:3d}| {r[0]:8d} {r[1]:8d} {r[2]:8d} | {r[3]:8d} {r[4]:8d} {r[5]:8d} {r[6]:8d} {r[7]:8d} |"
          f" {r[8]:8d} {r[9]:8d} {r[10]:8d} {r[11]:8d} {r[12]:8d} | {r[14]:8d} {r[15]:8d}")
mid = slice(n // 4, 3 * n // 4)
per = np.diff(T[mid, 1]).mean()
print(f"steady-state period (P0 ready to P0 ready): {per:.0f} cycles (ideal MMA-bound 2048 at D=128)")
for t, base in ((0, 3), (1, 8)):
    d = T[mid]
    print(f"tile{t}: wait S {np.mean(d[:, base+1]-d[:, base]):.0f}  ld {np.mean(d[:, base+2]-d[:, base+1]):.0f}  "
          f"max+exp {np.mean(d[:, base+3]-d[:, base+2]):.0f}  st+sig {np.mean(d[:, base+4]-d[:, base+3]):.0f}")
print(f"MMA wait for P0: {np.mean(T[mid,1]-T[mid,0]):.0f}   P0->P1: {np.mean(T[mid,2]-T[mid,1]):.0f}")
