"""Tiny K2 (tcgen05 verify, 2-CTA clusters) and K1 (head-packed draft) launches for
compute-sanitizer racecheck / synccheck (tools/gpu_sanitize.sh): small enough that the
instrumented run finishes in minutes.  Checks the outputs are finite."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_01278_b200 import kernels as K
from paper_2512_01278_b200.model import make_items
from paper_2512_01278_b200.paged import PagedKvPool

dev = torch.device("cuda")
d, Hkv, G, n, t, b = 128, 4, 4, 300, 5, 1
Hq = Hkv * G
pool = PagedKvPool(1, Hkv, d, 2 * 48, 16, b, 48, torch.bfloat16, dev)
for r in range(b):
    pool.ensure_tokens(r, n + t + 3)
pool.sync_table()
pool.k.normal_()
pool.v.normal_()
q = torch.randn(b * t, Hq, d, device=dev).to(torch.bfloat16)
out = torch.empty_like(q)
acc = torch.zeros(b * t, n + t, dtype=torch.int64, device=dev)
items = make_items([(r, r * t, t, n, 0, 0, 0, r * t, 1) for r in range(b)], dev)
K.attention(q, out, pool, 0, items, b, n + t, t, Hq, acc=acc, acc_row_stride=n + t, acc_shift=40)
torch.cuda.synchronize()
assert torch.isfinite(out.float()).all()
rng = np.random.default_rng(0)
bud = 60
crit = torch.from_numpy(np.stack([np.sort(rng.choice(n, bud, replace=False)) for _ in range(b)]).astype(np.int32)).to(dev)
ditems = make_items([(r, r, 1, n + 2, r * bud, bud, n, -1, 0) for r in range(b)], dev)
K.attention(q[:b], out[:b], pool, 0, ditems, b, bud + 3, 1, Hq, crit=crit)
torch.cuda.synchronize()
assert torch.isfinite(out.float()).all()
print("race_small ok")
