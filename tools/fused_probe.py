"""f3 diagnostics: one layer's verify launch (25 items, ctx 4608, k = 4) and draft launch
(103 items, 231 critical keys + 3 fresh) as two launches vs one fused launch (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_01278_b200 import kernels as K
from paper_2512_01278_b200.model import make_items
from paper_2512_01278_b200.paged import PagedKvPool
dev = torch.device("cuda")
Hkv, G, d, nq, n = 8, 4, 128, 5, 4608
Hq = Hkv * G
nv, nd, bud = int(os.environ.get("NV", 25)), int(os.environ.get("ND", 103)), 231
B = nv + nd
ppr = -(-(n + nq + 4) // 16)
pool = PagedKvPool(1, Hkv, d, ppr * B, 16, B, ppr, torch.bfloat16, dev)
for r in range(B): pool.ensure_tokens(r, n + nq + 4)
pool.sync_table(); pool.k.normal_(); pool.v.normal_()
rng = np.random.default_rng(0)
v_items = make_items([(r, r * nq, nq, n, 0, 0, 0, r * nq, 1) for r in range(nv)], dev)
crit = torch.from_numpy(np.stack([np.sort(rng.choice(n, bud, replace=False)) for _ in range(nd)]).astype(np.int32).reshape(-1)).to(dev)
d_items = make_items([(nv + i, nv * nq + i, 1, n + 2, i * bud, bud, n, -1, 0) for i in range(nd)], dev)
R = nv * nq + nd
q = torch.randn(R, Hq, d, device=dev).to(torch.bfloat16)
out = torch.zeros_like(q)
acc = torch.zeros(nv * nq, n + nq, dtype=torch.int64, device=dev)
v = dict(items=v_items, num_items=nv, max_keys=n + nq, max_nq=nq, acc=acc, acc_row_stride=n + nq, acc_shift=40)
dr = dict(items=d_items, num_items=nd, max_keys=bud + 3, crit=crit)
def sep():
    K.attention(q, out, pool, 0, v_items, nv, n + nq, nq, Hq, acc=acc, acc_row_stride=n + nq, acc_shift=40)
    K.attention(q, out, pool, 0, d_items, nd, bud + 3, 1, Hq, crit=crit)
def fused():
    assert K.attention_pair(q, out, pool, 0, v, dr, Hq)
def verify_only():
    K.attention(q, out, pool, 0, v_items, nv, n + nq, nq, Hq, acc=acc, acc_row_stride=n + nq, acc_shift=40)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for name, fn in (("verify only", verify_only), ("two launches", sep), ("fused", fused)):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); tot += e0.elapsed_time(e1)
    print(f"{name}: {tot / 10 * 1000:.1f} us")
