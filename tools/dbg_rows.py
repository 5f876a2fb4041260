import sys, torch, numpy as np
sys.path.insert(0, '.')
from tests import gpu_util as U
from paper_2511_12056_b200 import spa
for D, S, dist in ((96, 700, "D1"), (128, 700, "D1"), (96, 700, "D0"), (96, 256, "D1"), (96, 128, "D1")):
    q, k, v = U.qkv(1, S, 2, D, seed=3, dist=dist)
    o = spa.attention(q, k, v); torch.cuda.synchronize()
    ref = U.oracle_mha(q, k, v)
    err = np.abs(o.double().cpu().numpy() - ref)
    bad = err.max(axis=(2, 3)) > 2e-2          # [B, S]
    rows = np.nonzero(bad[0])[0]
    colerr = err[0].max(axis=(0, 1))
    print(D, S, dist, "bad rows", len(rows), rows[:10], "bad cols", np.nonzero(colerr > 2e-2)[0][:40], flush=True)
