"""Per-CTA phase breakdown of one K2 verify launch (diagnostics).
SD_ATTN_TRACE=1 python tools/trace_attn.py [ctx] [batch]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_01278_b200 import kernels as K, _native as N
from paper_2512_01278_b200.model import make_items
from paper_2512_01278_b200.paged import PagedKvPool
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4608
b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
d, Hkv, G, t = 128, 8, 4, 5
Hq = Hkv * G
dev = torch.device("cuda")
ppr = -(-(n + t) // 16)
pool = PagedKvPool(1, Hkv, d, ppr * b, 16, b, ppr, torch.bfloat16, dev)
for r in range(b):
    pool.ensure_tokens(r, n + t)
pool.sync_table()
pool.k.normal_(); pool.v.normal_()
q = torch.randn(b * t, Hq, d, device=dev).to(torch.bfloat16)
out = torch.empty_like(q)
items = make_items([(r, r * t, t, n, 0, 0, 0, r * t, 1) for r in range(b)], dev)
acc = torch.zeros(b * t, n + t, device=dev)
for _ in range(3):
    K.attention(q, out, pool, 0, items, b, n + t, t, Hq, acc=acc, acc_row_stride=n + t)
torch.cuda.synchronize()
lib = N.lib()
lib.sd_attention_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
nct = 8192
buf = np.zeros((nct, 8), dtype=np.uint64)
assert lib.sd_attention_trace(buf.ctypes.data, nct) == 0
buf = buf[buf[:, 0] > 0].astype(np.int64)
t0 = buf[:, 0].min()
rel = (buf - t0) / 1000.0
names = ["start", "setup", "phase1", "exchange", "phase2", "end"]
d = np.diff(rel[:, :6], axis=1)
print(f"ctas {len(buf)}  kernel span {rel[:,5].max():.1f} us")
for i in range(5):
    print(f"  {names[i]:>9s} -> {names[i+1]:<9s} mean {d[:, i].mean():7.2f} us  p90 {np.percentile(d[:, i], 90):7.2f}")
print(f"  cta lifetime mean {(rel[:,5]-rel[:,0]).mean():.2f} us; starts spread: first wave {np.sort(rel[:,0])[:148].max():.1f} us")
