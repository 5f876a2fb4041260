"""Run one attention case in a fresh process and report ok / error (debug helper).

    python tools/dbg_case.py D S dist [seed] [H]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from tests import gpu_util as U  # noqa: E402
from paper_2511_12056_b200 import spa  # noqa: E402

D, S, dist = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
seed = int(sys.argv[4]) if len(sys.argv) > 4 else 3
H = int(sys.argv[5]) if len(sys.argv) > 5 else 2
q, k, v = U.qkv(1, S, H, D, seed=seed, dist=dist)
try:
    out = spa.attention(q, k, v)
    torch.cuda.synchronize()
    ma, rl = U.errors(out, U.oracle_mha(q, k, v))
    print(f"D={D} S={S} {dist} seed={seed} H={H}: ok max_abs={ma:.2e} rel={rl:.2e}")
except Exception as e:
    print(f"D={D} S={S} {dist} seed={seed} H={H}: FAIL {str(e)[:100]}")
