"""Pin the CPU oracle (oracle/pillar_oracle.py) to the real reference.

Every expectation here was produced by the reference package itself
(tests/golden/make_golden.py); the oracle is only trusted because these pass.
"""

import numpy as np
import pytest

from oracle import pillar_oracle as O

C0_PLANTED = list(range(5, 256, 21))[:12]


def _weights(shp, planted=None):
    w = O.make_weights(O.Shape(*shp[:5], seed=shp[5]))
    return O.with_planted(w, planted) if planted else w


def test_weight_signatures(golden_weight_sigs):
    for key, sig in golden_weight_sigs.items():
        shp = tuple(int(x) for x in key.split("x"))
        w = _weights(shp)
        assert w.emb.ravel()[:8].tolist() == sig["emb_head"]
        assert float(w.emb.sum()) == sig["emb_sum"]
        for li, mats in enumerate(w.layer):
            for name, arr in mats.items():
                assert arr.ravel()[:4].tolist() == sig[f"L{li}.{name}.head"]
                assert float(arr.sum()) == sig[f"L{li}.{name}.sum"]


@pytest.mark.parametrize("tag,shp,planted", [
    ("tiny", (2, 4, 2, 8, 48, 0), None),
    ("c0", (2, 8, 2, 32, 512, 0), None),
    ("c0p", (2, 8, 2, 32, 512, 0), C0_PLANTED),
])
def test_forwards_match_reference(golden_forwards, tag, shp, planted):
    g = {k.split(".", 1)[1]: v for k, v in golden_forwards.items() if k.startswith(tag + ".")}
    w = _weights(shp, planted)
    toks = g["tokens"].tolist()
    kv = O.Kv(w.shape)
    lo, nk, nv, sc = O.full_forward(w, kv, toks[:-5])
    np.testing.assert_allclose(lo[-1], g["prefill_last_logits"], rtol=0, atol=1e-12)
    kv.push(nk, nv)
    lo2, nk2, nv2, sc2 = O.full_forward(w, kv, toks[-5:])
    np.testing.assert_allclose(lo2, g["verify_logits"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(nk2, g["verify_k"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(nv2, g["verify_v"], rtol=0, atol=1e-12)
    lse = np.stack([[s[1] for s in layer] for layer in sc2])
    np.testing.assert_allclose(lse, g["verify_lse"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(sc2[0][4][0], g["verify_logits_l0q4"], rtol=0, atol=1e-12)
    n_kv = len(kv)
    for a in (0, 2, 4):
        for fn in (O.importance, None):
            if fn is None:
                got = O.importance_grouped(sc2, n_kv + a + 1, a + 1, shp[1], shp[2])
            else:
                got = fn(sc2, n_kv + a + 1, a + 1, shp[1])
            np.testing.assert_allclose(got, g[f"importance_a{a}"], rtol=1e-12, atol=1e-15)
    imp = O.importance_grouped(sc, n_kv, len(toks) - 5, shp[1], shp[2])
    np.testing.assert_allclose(imp, g["prefill_importance"], rtol=1e-12, atol=1e-15)
    crit = O.topk_ascending(imp, O.budget_for(n_kv, 0.1))
    assert crit.tolist() == g["prefill_critical"].tolist()
    l1, ek, ev = O.sparse_forward(w, kv, crit, None, None, toks[-5])
    np.testing.assert_allclose(l1, g["sparse_logits1"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(ek, g["sparse_k1"], rtol=0, atol=1e-12)
    l2, _, _ = O.sparse_forward(w, kv, crit, ek[None], ev[None], int(np.argmax(l1)))
    np.testing.assert_allclose(l2, g["sparse_logits2"], rtol=0, atol=1e-12)


def test_budget_kats(golden_budgets):
    for n, s, b in golden_budgets:
        assert O.budget_for(n, s) == b
    assert O.budget_for(1000, 0.05) == 50
    assert O.budget_for(0, 0.5) == 1


def test_topk_kats(golden_topk):
    n = len([k for k in golden_topk if k.endswith(".values")])
    for i in range(n):
        v = golden_topk[f"t{i}.values"]
        b = int(golden_topk[f"t{i}.budget"])
        assert O.topk_ascending(v, b).tolist() == golden_topk[f"t{i}.positions"].tolist()
    # tie KATs (reference tests/test_selection.py:102-117)
    assert O.topk_ascending(np.array([5.0, 5.0, 5.0, 1.0]), 2).tolist() == [0, 1]
    assert O.topk_ascending(np.ones(9), 4).tolist() == [0, 1, 2, 3]
    assert O.topk_ascending(np.array([3.0, 1.0]), 10).tolist() == [0, 1]


def _run_case(c):
    w = _weights(tuple(c["shape"]), c["planted"])
    res = O.spec_decode(w, c["prompt"], c["out"], c["k"], c["s"], eos=c["eos"])
    return res


def test_token_streams_small(golden_streams):
    small = [c for c in golden_streams if c.get("tag") is None]
    assert len(small) >= 14
    for c in small:
        res = _run_case(c)
        assert res.tokens == c["tokens"]
        assert [[i, r.draft_target, r.accepted, r.kv_len, r.budget] for i, r in enumerate(res.rounds)] == c["rounds"]
        assert res.sparse_forwards == c["sparse_forwards"]
        assert res.full_forwards == c["full_forwards"]
        w = _weights(tuple(c["shape"]), c["planted"])
        assert O.greedy(w, c["prompt"], c["out"], eos=c["eos"]) == c["tokens"]


@pytest.mark.parametrize("tag", ["c0p", "c0"])
def test_token_stream_configs0(golden_streams, tag):
    c = [c for c in golden_streams if c.get("tag") == tag][0]
    res = _run_case(c)
    assert res.tokens == c["tokens"]
    assert res.alpha == c["alpha"]
