"""configs[4] kernel microbench: PillarAttn sparse draft (K1) and verify (K2)
attention over a paged bf16 KV cache, context 4K-64K, top-k 1-10%, k=2-8,
GQA 4/8, d=128 (BASELINE.json configs[4]).

    python bench_kernels.py [--ctx 4096,8192,...] [--batch 128] [--k 4] [--G 4] ...

One launch = one layer of a batch of requests.  Achieved GB/s = algorithmic
bytes (K/V rows touched, q/o, lse, score accumulator writes)
/ CUDA-event time, averaged over --iters launches after --warmup.  Before every
timed launch a 256 MB buffer is written (L2 flush, 2x the 126 MB L2) and a ~100 µs
device sleep keeps the GPU busy while the host enqueues the start event and the
launch, so the event pair brackets the kernel alone (no host launch path inside it; the
numbers did not move against the flush alone).
Prints one JSON line per shape.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", default="4096,8192,16384,32768,65536")
    ap.add_argument("--sparsity", default="0.01,0.05,0.10")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--G", type=int, default=4)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--only", default="both", choices=["both", "verify", "draft"])
    ap.add_argument("--shuffle-pages", action="store_true")
    args = ap.parse_args()

    import numpy as np
    import torch

    from paper_2512_01278_b200 import kernels as K
    from paper_2512_01278_b200.model import make_items
    from paper_2512_01278_b200.paged import PagedKvPool
    from paper_2512_01278_b200.selection import compute_budget

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    dev = torch.device("cuda")
    d, Hkv, G, B, k = 128, args.kv_heads, args.G, args.batch, args.k
    Hq = Hkv * G
    Pb = 2 * d * 2
    for n in [int(x) for x in args.ctx.split(",")]:
        # pool: B requests x (n + k + 1) tokens x layers; shrink batch so it fits ~120 GB
        per_req = (n + k + 1) * args.layers * Hkv * d * 2 * 2
        b = min(B, max(1, int(120e9 // per_req)))
        page = 16
        ppr = -(-(n + k + 1) // page)
        pool = PagedKvPool(args.layers, Hkv, d, ppr * b, page, b, ppr, torch.bfloat16, dev)
        if args.shuffle_pages:
            rng = np.random.default_rng(0)
            rng.shuffle(pool._free)
        for r in range(b):
            pool.ensure_tokens(r, n + k + 1)
        pool.sync_table()
        g = torch.Generator(device=dev)
        g.manual_seed(0)
        for l in range(args.layers):
            pool.k[l].copy_(torch.randn(pool.k[l].shape, generator=g, device=dev, dtype=torch.float32))
            pool.v[l].copy_(torch.randn(pool.v[l].shape, generator=g, device=dev, dtype=torch.float32))
        t = k + 1
        q = torch.randn(b * t, Hq, d, device=dev).to(torch.bfloat16)
        out = torch.empty_like(q)

        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

        def timeit(fn):
            for _ in range(args.warmup):
                fn(0)
            torch.cuda.synchronize()
            evs = []
            for i in range(args.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                flush.zero_()   # L2 flush
                # keep the GPU busy (~100 us) while the host enqueues e0 + the launch, so the
                # host-side launch path never shows up between the two events
                torch.cuda._sleep(200_000)
                e0.record()
                fn(i % args.layers)
                e1.record()
                evs.append((e0, e1))
            torch.cuda.synchronize()
            return sum(a.elapsed_time(bb) for a, bb in evs) / len(evs) / 1000.0

        if args.only in ("both", "verify"):
            items = make_items([(r, r * t, t, n, 0, 0, 0, r * t, 1) for r in range(b)], dev)
            W = n + t
            acc = torch.zeros(b * t, W, dtype=torch.int64, device=dev)
            shift = K.score_shift(1, 36, Hq)
            sec = timeit(lambda l: K.attention(q, out, pool, l, items, b, n + t, t, Hq, acc=acc, acc_row_stride=W,
                                               acc_shift=shift))
            byts = b * (Hkv * (n + t) * Pb + 2 * t * Hq * d * 2 + t * (n + t) * 8)
            flops = 4 * b * t * Hq * (n + t) * d
            print(json.dumps({"kernel": "K2 verify", "ctx": n, "batch": b, "k": k, "G": G, "us": sec * 1e6,
                              "GB/s": byts / sec / 1e9, "frac_hbm": byts / sec / 1e9 / hbm,
                              "TFLOP/s": flops / sec / 1e12}), flush=True)
            del acc
        if args.only in ("both", "draft"):
            for s in [float(x) for x in args.sparsity.split(",")]:
                bud = compute_budget(n, s)
                rng = np.random.default_rng(1)
                crit = np.stack([np.sort(rng.choice(n, size=bud, replace=False)) for _ in range(b)]).astype(np.int32)
                crit_d = torch.from_numpy(crit).to(dev)
                j = 2  # third draft of the round: fresh tail of 3 keys
                items = make_items([(r, r, 1, n + j, r * bud, bud, n, -1, 0) for r in range(b)], dev)
                qd = q[:b]
                od = out[:b]
                sec = timeit(lambda l: K.attention(qd, od, pool, l, items, b, bud + j + 1, 1, Hq, crit=crit_d))
                byts = b * (Hkv * (bud + j + 1) * Pb + 4 * bud + 2 * Hq * d * 2)
                print(json.dumps({"kernel": "K1 draft", "ctx": n, "sparsity": s, "budget": bud, "batch": b, "G": G,
                                  "us": sec * 1e6, "GB/s": byts / sec / 1e9, "frac_hbm": byts / sec / 1e9 / hbm}),
                      flush=True)
        del pool, q, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
