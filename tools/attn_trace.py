#!/usr/bin/env python
"""Per-iteration timeline of one attention CTA (debug build lib/libspa_trace.so, SPA_ATTN_TRACE).

    python -m paper_2511_12056_b200._build --trace
    SPA_LIB=paper_2511_12056_b200/lib/libspa_trace.so python tools/attn_trace.py [--D 128]
Events (clock64 cycles) per KV iteration j of CTA (0,0,0):
  TMA producer (lane 0):      11 K_j load issued   12 V_j load issued
  MMA issuer (elected lane):  2 K_j acquired -> QK(j) issued   10 V_j acquired
                              0 / 1  P(j) key-half 0 / 1 ready -> PV half issued
  softmax, lane 0 of the lane-quarter-0 warp of group j % NG:
                              3 loop top (before waiting for S(j))   4 S(j) ready   7 pass-1 max done
                              5 running max handed over              8 P half 0 released   6 P half 1 released
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
ap.add_argument("--rows", type=int, default=12)
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
n = min(256, (args.S + 127) // 128)
t0 = T[0, 2]
print("   j |  Kld    Vld   |  QKiss  Vacq   P0rdy   P1rdy |  top    Srdy   max    xchg   P0rel  P1rel")
mid0 = n // 2
for j in list(range(0, args.rows)) + list(range(mid0, mid0 + 6)) + list(range(n - 3, n)):
    r = T[j] - t0
    print(f"{j:4d} | {r[11]:7d} {r[12]:7d} | {r[2]:7d} {r[10]:7d} {r[0]:7d} {r[1]:7d} | {r[3]:7d} {r[4]:7d} {r[7]:7d} {r[5]:7d} {r[8]:7d} {r[6]:7d}")
js = np.arange(n // 4, 3 * n // 4)
d = T[js]
ideal = {128: 1024, 96: 768, 64: 512}[args.D]
print(f"steady-state period per KV tile: {np.diff(d[:, 1]).mean():.0f} cycles (P1 ready to P1 ready; "
      f"MMA-bound ideal {ideal} at D={args.D})")
print("per tile, mean cycles: "
      f"wait S {np.mean(d[:, 4] - d[:, 3]):.0f} | pass1 {np.mean(d[:, 7] - d[:, 4]):.0f} | "
      f"xchg {np.mean(d[:, 5] - d[:, 7]):.0f} | half0 {np.mean(d[:, 8] - d[:, 5]):.0f} | "
      f"half1 {np.mean(d[:, 6] - d[:, 8]):.0f} | softmax busy {np.mean(d[:, 6] - d[:, 4]):.0f}")
print(f"TMA latency (issue -> MMA warp sees data): K {np.mean(d[:, 2] - d[:, 11]):.0f}  V {np.mean(d[:, 10] - d[:, 12]):.0f}")
print("MMA side: "
      f"QK(j) issue -> P0(j) ready {np.mean(d[:, 0] - d[:, 2]):.0f} | P0 -> P1 {np.mean(d[:, 1] - d[:, 0]):.0f} | "
      f"S(j) ready - QK(j) issue {np.mean(d[:, 4] - d[:, 2]):.0f}")

# per-warp view (both CTAs of cluster 0, all four lane quarters): softmax duration S(j) seen -> P halves released
if hasattr(lib, "spa_debug_read_trace2"):
    buf2 = (ctypes.c_ulonglong * (256 * 8 * 3))()
    lib.spa_debug_read_trace2.argtypes = [ctypes.c_void_p]
    assert lib.spa_debug_read_trace2(ctypes.addressof(buf2)) == 0
    T2 = np.frombuffer(buf2, dtype=np.uint64).reshape(256, 8, 3).astype(np.int64)
    d2 = T2[js]
    print("per warp (CTA, quarter): mean S-seen -> 1st half / 2nd half released; leader S-seen offset vs quarter 0")
    for slot in range(8):
        c, q = divmod(slot, 4)
        off = np.mean(d2[:, slot, 0] - d2[:, 0, 0]) if c == 0 else float("nan")
        print(f"  cta {c} wq {q}: {np.mean(d2[:, slot, 1] - d2[:, slot, 0]):7.0f} {np.mean(d2[:, slot, 2] - d2[:, slot, 0]):7.0f}"
              f"   S offset {off:7.0f}")
