import sys, torch, numpy as np
sys.path.insert(0, '.')
from tests import gpu_util as U
from paper_2511_12056_b200 import spa
for D in (96, 128, 64):
    for S in (700, 2000):
        q, k, v = U.qkv(1, S, 2, D, seed=3, dist="D1")
        ref = U.oracle_mha(q, k, v)
        nbad = 0; nd = 0
        first = spa.attention(q, k, v); torch.cuda.synchronize()
        for it in range(40):
            o = spa.attention(q, k, v); torch.cuda.synchronize()
            if not torch.equal(o.view(torch.int16), first.view(torch.int16)): nd += 1
            err = np.abs(o.double().cpu().numpy() - ref).max()
            if err > 2e-2: nbad += 1
        print(D, S, "runs with error>2e-2:", nbad, "/40; runs differing from first:", nd, flush=True)
