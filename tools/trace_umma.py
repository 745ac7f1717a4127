"""Per-CTA phase breakdown of one tcgen05 attention launch (diagnostics).

    SD_ATTN_TRACE=1 python tools/trace_umma.py [ctx] [batch] [nq] [budget]

nq > 0: verify items (nq query tokens over ctx keys); nq = 0: draft items
(budget critical keys + 3 fresh).  Prints mean phase durations, CTA lifetime,
waves and the fraction of SM-time covered by at least one streaming CTA.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2512_01278_b200 import _native as N
from paper_2512_01278_b200 import kernels as K
from paper_2512_01278_b200.model import make_items
from paper_2512_01278_b200.paged import PagedKvPool

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 5
bud = int(sys.argv[4]) if len(sys.argv) > 4 else 205
d, Hkv, G = 128, 8, 4
Hq = Hkv * G
dev = torch.device("cuda")
t = max(nq, 1)
ppr = -(-(n + t + 3) // 16)
pool = PagedKvPool(1, Hkv, d, ppr * b, 16, b, ppr, torch.bfloat16, dev)
for r in range(b):
    pool.ensure_tokens(r, n + t + 3)
pool.sync_table()
pool.k.normal_()
pool.v.normal_()
q = torch.randn(b * t, Hq, d, device=dev).to(torch.bfloat16)
out = torch.empty_like(q)
if nq > 0:
    items = make_items([(r, r * t, t, n, 0, 0, 0, r * t, 1) for r in range(b)], dev)
    acc = torch.zeros(b * t, n + t, dtype=torch.int64, device=dev)
    run = lambda: K.attention(q, out, pool, 0, items, b, n + t, t, Hq, acc=acc, acc_row_stride=n + t, acc_shift=40)
else:
    rng = np.random.default_rng(0)
    crit = torch.from_numpy(np.stack([np.sort(rng.choice(n, bud, replace=False)) for _ in range(b)]).astype(np.int32)).to(dev)
    items = make_items([(r, r, 1, n + 2, r * bud, bud, n, -1, 0) for r in range(b)], dev)
    run = lambda: K.attention(q[:b], out[:b], pool, 0, items, b, bud + 3, 1, Hq, crit=crit)
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
lib = N.lib()
lib.sd_attention_trace_umma.argtypes = [ctypes.c_void_p, ctypes.c_int32]
ctas = 16384
buf = np.zeros((ctas, 12), dtype=np.uint64)
lib.sd_attention_trace_umma(buf.ctypes.data, ctas)
valid = buf[:, 0] > 0
tr = buf[valid].astype(np.int64)
t0 = tr[:, 0].min()
st = (tr[:, :8] - t0) / 1000.0  # us
names = ["setup", "phase1", "exchange", "phase2", "obar", "epilogue"]
durs = np.diff(st[:, :7], axis=1)
print(f"launch {ms * 1000:.1f} us, {valid.sum()} CTAs traced, span {(tr[:, 6].max() - t0) / 1000:.1f} us")
for i, nm in enumerate(names):
    print(f"  {nm:9s} mean {durs[:, i].mean():7.2f} us  p90 {np.percentile(durs[:, i], 90):7.2f}")
life = st[:, 6] - st[:, 0]
x8 = (tr[:, 8] - t0) / 1000.0
x10 = (tr[:, 10] - t0) / 1000.0
x11 = (tr[:, 11] - t0) / 1000.0
print(f"  exchange split: shuffles+bar {np.mean(x8 - st[:, 2]):.2f} us, cluster barrier+combine {np.mean(st[:, 3] - x8):.2f} us; "
      f"B1 arrivals after phase-1 end: MMA warp {np.mean(x10 - st[:, 2]):.2f} us, producer {np.mean(x11 - st[:, 2]):.2f} us")
print(f"  lifetime  mean {life.mean():7.2f} us; producer done at {np.mean(st[:, 7] - st[:, 0]):.2f} us after start")
smid = (tr[:, 9] & 0xffffffff).astype(np.int64)
tiles = (tr[:, 9] >> 32).astype(np.int64)
print(f"  tiles per CTA mean {tiles.mean():.2f}; SMs used {len(np.unique(smid))}; CTAs per SM {len(tr) / len(np.unique(smid)):.1f}")
# coverage: fraction of [0, span] per SM with >= 1 CTA in phase1..phase2 (streaming)
span = st[:, 6].max()
grid = np.linspace(0, span, 2000)
cov1 = cov2 = 0.0
for s in np.unique(smid):
    m = smid == s
    a = ((grid[None, :] >= st[m, 1][:, None]) & (grid[None, :] < st[m, 4][:, None])).sum(axis=0)
    cov1 += (a >= 1).mean()
    cov2 += (a >= 2).mean()
ns = len(np.unique(smid))
print(f"  SM-time with >=1 CTA streaming {cov1 / ns:.2f}, with 2 {cov2 / ns:.2f}")
# max CTAs alive at once on one SM (start..end overlap)
mx = 0
for s_ in np.unique(smid):
    m = smid == s_
    ev = sorted([(a, 1) for a in st[m, 0]] + [(b, -1) for b in st[m, 6]], key=lambda x: (x[0], x[1]))
    cur = 0
    for _, dlt in ev:
        cur += dlt
        mx = max(mx, cur)
print(f"  max CTAs alive on one SM: {mx}")
