"""Generate the golden fixtures that pin ``oracle/pillar_oracle.py``.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports the reference package read-only under the alias ``spardec_ref``
and records, from the REFERENCE itself (not from our oracle):

  * weight signatures of ``init_model``                       (model.py:171-195)
  * forward_full logits / lse / importance, forward_sparse logits
                                                            (model.py:290-385)
  * budget and top-k known answers                           (selection.py:167-204)
  * token streams + round records of decode_to_completion and greedy_decode,
    including the configs[0] shape (L=2, Hq=8, Hkv=2, d=32, V=512, 4 requests
    x 256-token prompt x 1024 output tokens, k=4, s=0.05), random-init and
    planted                                                   (engine.py:154-298)

The fixtures are small (npz / json) and committed; the GPU box never reads
/root/reference.
"""

from __future__ import annotations

import importlib.util
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src/spardec"
OUT = Path(__file__).resolve().parent


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "spardec_ref", f"{REF}/__init__.py", submodule_search_locations=[REF]
    )
    mod = importlib.util.module_from_spec(spec)
    sys.modules["spardec_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def sim_prompt(seed, rid, n, vocab):
    g = np.random.default_rng(np.random.SeedSequence([seed, rid]))
    return g.integers(0, vocab, size=n).tolist()


C0_PLANTED = list(range(5, 256, 21))[:12]


def main() -> None:
    load_reference()
    from spardec_ref import engine as RE
    from spardec_ref import model as RM
    from spardec_ref import selection as RS

    # -- weights ---------------------------------------------------------------
    sigs = {}
    for shp in [(2, 4, 2, 8, 48, 0), (2, 8, 2, 32, 512, 0), (1, 4, 4, 16, 40, 7)]:
        m = RM.init_model(RM.ModelConfig(*shp[:5], seed=shp[5]))
        entry = {"emb_head": m.embedding.ravel()[:8].tolist(), "emb_sum": float(m.embedding.sum())}
        for li, lw in enumerate(m.layers):
            for name in ("mlp_in", "mlp_out", "wk", "wo", "wq", "wv"):
                arr = getattr(lw, name)
                entry[f"L{li}.{name}.head"] = arr.ravel()[:4].tolist()
                entry[f"L{li}.{name}.sum"] = float(arr.sum())
        sigs["x".join(map(str, shp))] = entry
    (OUT / "weights_sig.json").write_text(json.dumps(sigs, indent=1))

    # -- forwards ----------------------------------------------------------------
    arrays = {}
    for tag, shp, planted in [("tiny", (2, 4, 2, 8, 48, 0), None),
                              ("c0", (2, 8, 2, 32, 512, 0), None),
                              ("c0p", (2, 8, 2, 32, 512, 0), C0_PLANTED)]:
        cfg = RM.ModelConfig(*shp[:5], seed=shp[5])
        model = RM.init_model(cfg)
        if planted:
            model = RM.plant_attention_concentration(model, planted)
        n_prompt = 40 if tag == "tiny" else 300
        toks = sim_prompt(11, 0, n_prompt, shp[4])
        cache = RM.KvCache(cfg)
        rows, entries, log = RM.forward_full(model, cache, toks[:-5])
        cache.extend(entries)
        rows2, entries2, log2 = RM.forward_full(model, cache, toks[-5:])
        arrays[f"{tag}.tokens"] = np.asarray(toks)
        arrays[f"{tag}.prefill_last_logits"] = rows[-1]
        arrays[f"{tag}.verify_logits"] = np.stack(rows2)
        arrays[f"{tag}.verify_k"] = np.stack([e.k for e in entries2])
        arrays[f"{tag}.verify_v"] = np.stack([e.v for e in entries2])
        arrays[f"{tag}.verify_lse"] = np.stack([[r.lse for r in lr] for lr in log2.layers])
        arrays[f"{tag}.verify_logits_l0q4"] = log2.layers[0][4].logits
        n_kv = len(cache)
        for a in (0, 2, 4):
            imp = RS.importance_from_log(log2.slice_queries(a + 1), n_kv + a + 1)
            arrays[f"{tag}.importance_a{a}"] = imp
        imp_p = RS.importance_from_log(log, n_kv)
        arrays[f"{tag}.prefill_importance"] = imp_p
        b = RS.compute_budget(n_kv, 0.1)
        crit = RS.select_critical_tokens(imp_p, b)
        arrays[f"{tag}.prefill_critical"] = crit.positions
        # sparse draft: two steps over the critical set with one fresh entry
        l1, e1 = RM.forward_sparse(model, cache, crit, [], toks[-5])
        l2, _ = RM.forward_sparse(model, cache, crit, [e1], int(np.argmax(l1)))
        arrays[f"{tag}.sparse_logits1"] = l1
        arrays[f"{tag}.sparse_logits2"] = l2
        arrays[f"{tag}.sparse_k1"] = e1.k
    np.savez_compressed(OUT / "forwards.npz", **arrays)

    # -- selection KATs ------------------------------------------------------------
    rng = np.random.default_rng(7)
    budgets = []
    for _ in range(400):
        n = int(rng.integers(0, 70000))
        s = float(rng.choice([0.01, 0.02, 0.05, 0.07, 0.1, 0.25, 1.0, float(rng.uniform(1e-4, 1))]))
        budgets.append([n, s, RS.compute_budget(n, s)])
    budgets += [[1000, 0.05, RS.compute_budget(1000, 0.05)], [560, 0.07, RS.compute_budget(560, 0.07)]]
    topk = {}
    for i in range(60):
        n = int(rng.integers(1, 3000))
        v = rng.normal(size=n)
        if i % 3 == 0:
            v = np.round(v, 1)
        if i % 5 == 0:
            v = np.abs(np.round(v, 0))
        b = int(rng.integers(1, n + 3))
        topk[f"t{i}.values"] = v
        topk[f"t{i}.budget"] = np.asarray(b)
        topk[f"t{i}.positions"] = RS.select_critical_tokens(v, b).positions
    (OUT / "budget_kat.json").write_text(json.dumps(budgets))
    np.savez_compressed(OUT / "topk_kat.npz", **topk)

    # -- token streams ---------------------------------------------------------------
    streams = []
    cases = []
    crng = np.random.default_rng(20260818)
    for i in range(12):
        shp = (int(crng.integers(1, 3)), 4, 2, 8, int(crng.integers(24, 65)), int(crng.integers(0, 2**31)))
        cases.append(dict(shape=shp, prompt_len=int(crng.integers(4, 33)), k=int(crng.integers(1, 9)),
                          s=float(crng.uniform(0.02, 1.0)) if i % 4 else 1.0,
                          out=int(crng.integers(16, 97)), planted=None, eos_from=None))
    cases.append(dict(shape=(2, 4, 2, 8, 48, 5), prompt_len=12, k=4, s=0.3, out=48, planted=None, eos_from=20))
    cases.append(dict(shape=(2, 4, 2, 8, 48, 1), prompt_len=20, k=4, s=0.25, out=32, planted=[2, 7, 11], eos_from=None))
    for rid in range(4):
        cases.append(dict(shape=(2, 8, 2, 32, 512, 0), prompt_len=256, k=4, s=0.05, out=1024,
                          planted=None, eos_from=None, rid=rid, tag="c0"))
    for rid in range(4):
        cases.append(dict(shape=(2, 8, 2, 32, 512, 0), prompt_len=256, k=4, s=0.05, out=1024,
                          planted=C0_PLANTED, eos_from=None, rid=rid, tag="c0p"))
    for ci, c in enumerate(cases):
        t0 = time.time()
        shp = c["shape"]
        model = RM.init_model(RM.ModelConfig(*shp[:5], seed=shp[5]))
        if c["planted"]:
            model = RM.plant_attention_concentration(model, c["planted"])
        prompt = sim_prompt(0, c.get("rid", ci), c["prompt_len"], shp[4])
        eos = None
        if c["eos_from"] is not None:
            eos = RE.greedy_decode(model, prompt, c["out"])[c["eos_from"]]
        req = RE.DecodeRequest(request_id=ci, prompt=prompt, max_output=c["out"], eos_token=eos)
        committed, stats = RE.decode_to_completion(model, req, c["k"], c["s"])
        g = RE.greedy_decode(model, prompt, c["out"], eos_token=eos)
        assert g == committed
        streams.append(dict(c, prompt=prompt, eos=eos, tokens=committed,
                            rounds=[list(r) for r in stats.csv_rows()],
                            sparse_forwards=stats.sparse_forwards, full_forwards=stats.full_forwards,
                            alpha=stats.realized_alpha))
        print(f"case {ci} shape={shp} out={c['out']} alpha={stats.realized_alpha:.3f} {time.time()-t0:.1f}s")
    (OUT / "streams.json").write_text(json.dumps(streams))


def offload_streams() -> None:
    """The REFERENCE's token-level serving loop under KV offload pressure (OFFLOAD policy,
    120-page pool, 16-page chunks; simulate.py:535, kvpool.py:213-237,272-311): its per-request
    outputs are the golden streams of tests/test_serving_gpu.py's offload test."""
    load_reference()
    from spardec_ref import kvpool as RK
    from spardec_ref import model as RM
    from spardec_ref import simulate as RSim
    from spardec_ref import workload as RW

    out = []
    for seed, n, inp, outl, cap in [(0, 4, 16, 24, 120), (0, 6, 20, 40, 160)]:
        wl = RW.WorkloadSpec(n_requests=n, input_len=RW.LengthSpec(RW.LengthDist.CONSTANT, inp),
                             output_len=RW.LengthSpec(RW.LengthDist.CONSTANT, outl), seed=seed)
        mc = RM.ModelConfig(2, 4, 2, 8, 48, seed=0)
        rep = RSim.run_token_sim(wl, mc, RSim.SimConfig(k=3, alpha=0.0, sparsity=0.4, max_batch=n),
                                 RSim.KvPoolConfig(capacity_pages=cap, page_bytes=64, chunk_pages=16,
                                                   policy=RK.KvPolicy.OFFLOAD))
        out.append(dict(seed=seed, n=n, input_len=inp, output_len=outl, capacity=cap,
                        outputs={str(k): v for k, v in rep.outputs.items()},
                        max_offloaded=max(r.offloaded_pages for r in rep.iterations)))
        print(f"offload case n={n} cap={cap}: max offloaded pages {out[-1]['max_offloaded']}")
    (OUT / "offload_streams.json").write_text(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1:] == ["offload"]:
        offload_streams()
        raise SystemExit(0)
    main()
