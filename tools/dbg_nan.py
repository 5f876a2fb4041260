import sys, torch
sys.path.insert(0, '.')
from tests import gpu_util as U
from paper_2511_12056_b200 import spa
for D in (64, 96, 128):
    for S in (128, 200, 256, 300, 384, 1000):
        q, k, v = U.qkv(1, S, 1, D, seed=S + D)
        o = spa.attention(q, k, v); torch.cuda.synchronize()
        bad = torch.isnan(o.float())
        rows = bad.any(-1).any(-1).nonzero().flatten().tolist()
        ref = U.oracle_mha(q, k, v)
        ma, rl = U.errors(o, ref) if not bad.any() else (float('nan'), float('nan'))
        print(D, S, "nan rows:", len(rows), rows[:5], rows[-3:] if rows else [], "err", ma, rl, flush=True)
