import sys, torch, numpy as np
sys.path.insert(0, '.')
from tests import gpu_util as U
from paper_2511_12056_b200 import spa
for dist in ("D0", "D1", "D4"):
    for D, S in ((128, 2000), (64, 700)):
        q, k, v = U.qkv(1, S, 2, D, seed=3, dist=dist)
        ref = U.oracle_mha(q, k, v)
        nbad = 0; nd = 0; worst = 0
        first = spa.attention(q, k, v); torch.cuda.synchronize()
        for it in range(20):
            o = spa.attention(q, k, v); torch.cuda.synchronize()
            if not torch.equal(o.view(torch.int16), first.view(torch.int16)): nd += 1
            err = np.abs(o.double().cpu().numpy() - ref)
            worst = max(worst, err.max())
            if err.max() > 2e-2: nbad += 1
        bad_rows = np.nonzero(err.max(axis=(0, 2, 3)) > 2e-2)[0]
        print(dist, D, S, "bad runs", nbad, "/20 differing", nd, "worst", worst, "bad rows(last)", bad_rows[:12], flush=True)
