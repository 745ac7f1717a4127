"""Kernel-level parity on the B200 (calls go through the C ABI).

Oracles: oracle/pillar_oracle.attend_one (fp64 restatement of model.py:229-253,
pinned to the reference) for attention outputs / lse; the reference's own
golden top-k / budget known answers; numpy for argmax / accept.
Tolerances (north_star): attention 1e-4 in fp32 mode, 2e-2 max-abs in bf16.
"""

import math

import numpy as np
import pytest
import torch

from oracle import pillar_oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2512_01278_b200 import kernels as K  # noqa: E402
from paper_2512_01278_b200.model import make_items  # noqa: E402
from paper_2512_01278_b200.paged import PagedKvPool  # noqa: E402

DEV = torch.device("cuda")


def _acc(rows, width, Hq, L=1):
    """Zeroed fixed-point score accumulators and their shift (one row per query token)."""
    return torch.zeros(rows, width, dtype=torch.int64, device=DEV), K.score_shift(1, L, Hq)


def _accf(acc, shift):
    return K.scores_to_float(acc, shift).cpu().numpy()


def _pool(L, Hkv, d, n_tokens, rows, dtype, page=16, shuffle_seed=None):
    pages_per_row = -(-n_tokens // page)
    pool = PagedKvPool(L, Hkv, d, pages_per_row * rows + 3, page, rows, pages_per_row, dtype, DEV)
    if shuffle_seed is not None:  # scatter physical pages to stress the gather path
        rng = np.random.default_rng(shuffle_seed)
        rng.shuffle(pool._free)
    for r in range(rows):
        pool.ensure_tokens(r, n_tokens)
    pool.sync_table()
    return pool


def _fill(pool, row, n, rng, scale=1.0):
    L, Hkv, d = pool.layers, pool.kv_heads, pool.head_dim
    k = rng.normal(size=(n, L, Hkv, d)) * scale
    v = rng.normal(size=(n, L, Hkv, d))
    pool.write(row, range(n), torch.from_numpy(k), torch.from_numpy(v))
    return k, v


def _ref_rows(q, k, v, Hq, Hkv, d, crit, dense, qpos0, planted=(), bonus=0.0):
    """Per query token: oracle attend_one over crit U dense[:qpos+1] (dtype-rounded inputs)."""
    shape = O.Shape(1, Hq, Hkv, d, 2)
    outs, lses, accs = [], [], []
    for t in range(q.shape[0]):
        pos_list = list(crit) + [p for p in dense if p <= qpos0 + t]
        keys = k[pos_list]
        vals = v[pos_list]
        bias = None
        if planted:
            bias = np.where(np.isin(pos_list, planted), bonus, 0.0)
        ctx, lg, lse = O.attend_one(q[t], keys, vals, shape, bias)
        outs.append(ctx.reshape(Hq, d))
        lses.append(lse)
        p = np.exp(lg - lse[:, None]).sum(axis=0)
        accs.append(dict(zip(pos_list, p)))
    return np.stack(outs), np.stack(lses), accs


@pytest.mark.parametrize("dtype,force_generic,d,G", [
    (torch.float32, True, 32, 4), (torch.float32, True, 8, 2), (torch.bfloat16, False, 128, 4),
    (torch.bfloat16, False, 128, 8), (torch.bfloat16, False, 64, 4), (torch.bfloat16, True, 128, 4),
])
def test_verify_attention_matches_oracle(dtype, force_generic, d, G):
    rng = np.random.default_rng(0)
    Hkv, L = 2, 2
    Hq = Hkv * G
    n0, nq = 700, 5
    pool = _pool(L, Hkv, d, n0 + nq, 2, dtype, shuffle_seed=1)
    k, v = _fill(pool, 1, n0 + nq, rng)
    kr, vr = pool.read(1, range(n0 + nq))
    kr, vr = kr.double().cpu().numpy(), vr.double().cpu().numpy()
    q = torch.from_numpy(rng.normal(size=(nq, Hq, d))).to(DEV, dtype)
    out = torch.empty_like(q)
    lse = torch.empty(nq, Hq, dtype=torch.float32, device=DEV)
    acc, shift = _acc(nq, n0 + nq, Hq)
    items = make_items([(1, 0, nq, n0, 0, 0, 0, 0, 1)], DEV)
    planted = torch.tensor([3, 77, 400], dtype=torch.int32, device=DEV)
    for use_planted in (False, True):
        acc.zero_()
        K.attention(q, out, pool, 1, items, 1, n0 + nq, nq, Hq, lse=lse, acc=acc, acc_row_stride=n0 + nq,
                    acc_shift=shift,
                    planted=planted if use_planted else None, planted_bonus=3.0 if use_planted else 0.0,
                    force_generic=force_generic)
        torch.cuda.synchronize()
        ro, rl, ra = _ref_rows(q.double().cpu().numpy(), kr[:, 1], vr[:, 1], Hq, Hkv, d, [], range(n0 + nq), n0,
                               planted=(3, 77, 400) if use_planted else (), bonus=3.0)
        tol = 1e-4 if dtype == torch.float32 else 2e-2
        assert np.abs(out.double().cpu().numpy() - ro).max() <= tol
        assert np.abs(lse.double().cpu().numpy() - rl).max() <= (1e-4 if dtype == torch.float32 else 2e-2)
        acc_h = _accf(acc, shift)
        for t in range(nq):
            want = np.zeros(n0 + nq)
            for p_, val in ra[t].items():
                want[p_] = val
            assert np.abs(acc_h[t] - want).max() <= (1e-5 if dtype == torch.float32 else 2e-2 * G)
            if n0 + t + 1 < acc_h.shape[1]:
                assert acc_h[t, n0 + t + 1:].max() == 0.0  # causally hidden tail carries exactly zero


@pytest.mark.parametrize("dtype,force_generic,d", [
    (torch.float32, True, 32), (torch.bfloat16, False, 128), (torch.bfloat16, False, 64)])
def test_sparse_draft_attention_matches_oracle(dtype, force_generic, d):
    rng = np.random.default_rng(1)
    Hkv, G, L = 4, 4, 1
    Hq = Hkv * G
    n0, j = 3000, 2
    pool = _pool(L, Hkv, d, n0 + j + 1, 1, dtype, shuffle_seed=3)
    _fill(pool, 0, n0 + j + 1, rng)
    kr, vr = pool.read(0, range(n0 + j + 1))
    kr, vr = kr.double().cpu().numpy()[:, 0], vr.double().cpu().numpy()[:, 0]
    crit = np.sort(rng.choice(n0, size=151, replace=False)).astype(np.int32)
    crit_dev = torch.from_numpy(crit).to(DEV)
    q = torch.from_numpy(rng.normal(size=(1, Hq, d))).to(DEV, dtype)
    out = torch.empty_like(q)
    lse = torch.empty(1, Hq, dtype=torch.float32, device=DEV)
    items = make_items([(0, 0, 1, n0 + j, 0, len(crit), n0, -1, 0)], DEV)
    K.attention(q, out, pool, 0, items, 1, len(crit) + j + 1, 1, Hq, crit=crit_dev, lse=lse,
                force_generic=force_generic)
    torch.cuda.synchronize()
    ro, rl, _ = _ref_rows(q.double().cpu().numpy(), kr, vr, Hq, Hkv, d, crit.tolist(), range(n0, n0 + j + 1), n0 + j)
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    assert np.abs(out.double().cpu().numpy() - ro).max() <= tol
    assert np.abs(lse.double().cpu().numpy() - rl).max() <= tol


@pytest.mark.parametrize("G,use_planted,buds,Hkv", [(4, True, (37, 130, 200), 8), (8, False, (37, 130, 200), 8),
                                                    (8, True, (37, 130, 200), 8), (4, True, (300, 700, 900), 8),
                                                    (8, False, (250, 500, 900), 8), (4, False, (10, 26, 29), 2),
                                                    (8, True, (5, 20, 60), 8), (4, True, (3, 300, 900), 2)])
def test_draft_attention_head_packed_bf16(G, use_planted, buds, Hkv):
    """Draft items of several requests (kv heads packed per CTA, block-diagonal P): outputs and
    lse per request vs the oracle over critical U fresh U self, with the planted bias. The
    larger budgets exceed the 4-head packing's resident logits and take the 2-head, 64-key-tile
    variant."""
    rng = np.random.default_rng(20 + G)
    d, B = 128, 3
    Hq = Hkv * G
    n0 = 2000
    pool = _pool(1, Hkv, d, n0 + 4, B, torch.bfloat16, shuffle_seed=7)
    for r in range(B):
        _fill(pool, r, n0 + 4, rng)
    js = [0, 1, 3]
    crit = [np.sort(rng.choice(n0, size=b, replace=False)).astype(np.int32) for b in buds]
    planted = np.array(sorted(set(int(x) for x in crit[1][:3]) | {n0 + 1}), dtype=np.int32)
    offs = np.cumsum([0] + list(buds))
    crit_dev = torch.from_numpy(np.concatenate(crit)).to(DEV)
    q = torch.from_numpy(rng.normal(size=(B, Hq, d))).to(DEV, torch.bfloat16)
    # one sentinel row past the outputs: no write may land outside the items' rows
    out_all = torch.full((B + 1, Hq, d), 7.0, dtype=torch.bfloat16, device=DEV)
    lse_all = torch.full((B + 1, Hq), 7.0, dtype=torch.float32, device=DEV)
    out, lse = out_all[:B], lse_all[:B]
    items = make_items([(r, r, 1, n0 + js[r], int(offs[r]), buds[r], n0, -1, 0) for r in range(B)], DEV)
    K.attention(q, out, pool, 0, items, B, max(b + j + 1 for b, j in zip(buds, js)), 1, Hq, crit=crit_dev, lse=lse,
                planted=torch.from_numpy(planted).to(DEV) if use_planted else None,
                planted_bonus=2.5 if use_planted else 0.0)
    torch.cuda.synchronize()
    assert bool((out_all[B] == 7.0).all()) and bool((lse_all[B] == 7.0).all())
    for r in range(B):
        kr, vr = pool.read(r, range(n0 + 4))
        kr, vr = kr.double().cpu().numpy()[:, 0], vr.double().cpu().numpy()[:, 0]
        ro, rl, _ = _ref_rows(q[r:r + 1].double().cpu().numpy(), kr, vr, Hq, Hkv, d, crit[r].tolist(),
                              range(n0, n0 + js[r] + 1), n0 + js[r],
                              planted=tuple(planted.tolist()) if use_planted else (), bonus=2.5)
        assert np.abs(out[r:r + 1].double().cpu().numpy() - ro).max() <= 2e-2
        assert np.abs(lse[r:r + 1].double().cpu().numpy() - rl).max() <= 2e-2


def test_batched_items_mixed_lengths_bf16():
    """Many items of ragged length in one launch (cluster split > 1)."""
    rng = np.random.default_rng(5)
    Hkv, G, d, L = 8, 4, 128, 1
    Hq = Hkv * G
    lens = [1, 63, 64, 65, 1000, 4099, 8709]
    nq = 5
    pool = _pool(L, Hkv, d, max(lens) + nq, len(lens), torch.bfloat16, shuffle_seed=9)
    for r, n in enumerate(lens):
        _fill(pool, r, n + nq, rng)
    rows = [(r, r * nq, nq, n, 0, 0, 0, r * nq, 1) for r, n in enumerate(lens)]
    items = make_items(rows, DEV)
    q = torch.from_numpy(rng.normal(size=(len(lens) * nq, Hq, d))).to(DEV, torch.bfloat16)
    out = torch.empty_like(q)
    lse = torch.empty(len(lens) * nq, Hq, dtype=torch.float32, device=DEV)
    W = max(lens) + nq
    acc, shift = _acc(len(lens) * nq, W, Hq)
    K.attention(q, out, pool, 0, items, len(lens), max(lens) + nq, nq, Hq, lse=lse, acc=acc, acc_row_stride=W,
                acc_shift=shift)
    torch.cuda.synchronize()
    for r, n in enumerate(lens):
        kr, vr = pool.read(r, range(n + nq))
        kr, vr = kr.double().cpu().numpy()[:, 0], vr.double().cpu().numpy()[:, 0]
        qs = q[r * nq:(r + 1) * nq].double().cpu().numpy()
        ro, rl, ra = _ref_rows(qs, kr, vr, Hq, Hkv, d, [], range(n + nq), n)
        assert np.abs(out[r * nq:(r + 1) * nq].double().cpu().numpy() - ro).max() <= 2e-2
        assert np.abs(lse[r * nq:(r + 1) * nq].double().cpu().numpy() - rl).max() <= 2e-2
        a = _accf(acc[r * nq:(r + 1) * nq], shift)
        # each query's probabilities sum to 1 per q head: Hq in total
        np.testing.assert_allclose(a.sum(axis=1), Hq * np.ones(nq), rtol=2e-2)
        for t in range(nq):
            want = np.zeros(W)
            for p_, val in ra[t].items():
                want[p_] = val
            assert np.abs(a[t] - want).max() <= 2e-2


@pytest.mark.parametrize("n0,G,nq", [(30000, 4, 5), (12000, 8, 3), (64000, 4, 2)])
def test_verify_attention_long_context_bf16(n0, G, nq):
    """Contexts past the TMEM-resident capacity of a 16-CTA cluster: evicted tiles are
    recomputed in phase 2 (K re-read); outputs, lse and scores must not change."""
    rng = np.random.default_rng(n0)
    Hkv, d = 2, 128
    Hq = Hkv * G
    pool = _pool(1, Hkv, d, n0 + nq, 1, torch.bfloat16, shuffle_seed=4)
    _fill(pool, 0, n0 + nq, rng, scale=0.5)
    kr, vr = pool.read(0, range(n0 + nq))
    kr, vr = kr.double().cpu().numpy()[:, 0], vr.double().cpu().numpy()[:, 0]
    q = torch.from_numpy(rng.normal(size=(nq, Hq, d))).to(DEV, torch.bfloat16)
    out = torch.empty_like(q)
    lse = torch.empty(nq, Hq, dtype=torch.float32, device=DEV)
    W = n0 + nq
    acc, shift = _acc(nq, W, Hq)
    items = make_items([(0, 0, nq, n0, 0, 0, 0, 0, 1)], DEV)
    K.attention(q, out, pool, 0, items, 1, n0 + nq, nq, Hq, lse=lse, acc=acc, acc_row_stride=W, acc_shift=shift)
    torch.cuda.synchronize()
    ro, rl, ra = _ref_rows(q.double().cpu().numpy(), kr, vr, Hq, Hkv, d, [], range(n0 + nq), n0)
    assert np.abs(out.double().cpu().numpy() - ro).max() <= 2e-2
    assert np.abs(lse.double().cpu().numpy() - rl).max() <= 2e-2
    a = _accf(acc, shift)
    np.testing.assert_allclose(a.sum(axis=1), Hq * np.ones(nq), rtol=2e-2)
    for t in range(nq):
        want = np.zeros(W)
        for p_, val in ra[t].items():
            want[p_] = val
        assert np.abs(a[t] - want).max() <= 2e-2


def test_sparse_draft_attention_large_budget_bf16():
    """10% of a 64K context (6.4K critical keys + fresh tail) in one draft item."""
    rng = np.random.default_rng(11)
    Hkv, G, d = 2, 4, 128
    Hq = Hkv * G
    n0, j = 64000, 3
    pool = _pool(1, Hkv, d, n0 + j + 1, 1, torch.bfloat16, shuffle_seed=6)
    _fill(pool, 0, n0 + j + 1, rng, scale=0.5)
    kr, vr = pool.read(0, range(n0 + j + 1))
    kr, vr = kr.double().cpu().numpy()[:, 0], vr.double().cpu().numpy()[:, 0]
    crit = np.sort(rng.choice(n0, size=6400, replace=False)).astype(np.int32)
    q = torch.from_numpy(rng.normal(size=(1, Hq, d))).to(DEV, torch.bfloat16)
    out = torch.empty_like(q)
    lse = torch.empty(1, Hq, dtype=torch.float32, device=DEV)
    items = make_items([(0, 0, 1, n0 + j, 0, len(crit), n0, -1, 0)], DEV)
    K.attention(q, out, pool, 0, items, 1, len(crit) + j + 1, 1, Hq, crit=torch.from_numpy(crit).to(DEV), lse=lse)
    torch.cuda.synchronize()
    ro, rl, _ = _ref_rows(q.double().cpu().numpy(), kr, vr, Hq, Hkv, d, crit.tolist(), range(n0, n0 + j + 1), n0 + j)
    assert np.abs(out.double().cpu().numpy() - ro).max() <= 2e-2
    assert np.abs(lse.double().cpu().numpy() - rl).max() <= 2e-2


def test_verify_mixed_token_counts_short_contexts_bf16():
    """One launch mixing 1..5-token verify items (first-round round targets) over short
    contexts (0 .. 1000 committed keys, tile and page boundaries), planted bias on."""
    rng = np.random.default_rng(21)
    Hkv, G, d = 8, 4, 128
    Hq = Hkv * G
    cases = [(0, 2), (1, 5), (127, 3), (128, 1), (129, 5), (1000, 4)]  # (n0, tokens)
    maxn = max(n + t for n, t in cases)
    pool = _pool(1, Hkv, d, maxn, len(cases), torch.bfloat16, shuffle_seed=13)
    for r, (n, t) in enumerate(cases):
        _fill(pool, r, n + t, rng)
    rows, q0 = [], 0
    for r, (n, t) in enumerate(cases):
        rows.append((r, q0, t, n, 0, 0, 0, r * 5, 1))
        q0 += t
    items = make_items(rows, DEV)
    q = torch.from_numpy(rng.normal(size=(q0, Hq, d))).to(DEV, torch.bfloat16)
    out = torch.empty_like(q)
    lse = torch.empty(q0, Hq, dtype=torch.float32, device=DEV)
    acc, shift = _acc(len(cases) * 5, maxn, Hq)
    planted = (5, 128, 1001)
    K.attention(q, out, pool, 0, items, len(cases), maxn, 5, Hq, lse=lse, acc=acc, acc_row_stride=maxn,
                acc_shift=shift,
                planted=torch.tensor(planted, dtype=torch.int32, device=DEV), planted_bonus=1.5)
    torch.cuda.synchronize()
    q0 = 0
    for r, (n, t) in enumerate(cases):
        kr, vr = pool.read(r, range(n + t))
        kr, vr = kr.double().cpu().numpy()[:, 0], vr.double().cpu().numpy()[:, 0]
        qs = q[q0:q0 + t].double().cpu().numpy()
        ro, rl, ra = _ref_rows(qs, kr, vr, Hq, Hkv, d, [], range(n + t), n, planted=planted, bonus=1.5)
        assert np.abs(out[q0:q0 + t].double().cpu().numpy() - ro).max() <= 2e-2
        assert np.abs(lse[q0:q0 + t].double().cpu().numpy() - rl).max() <= 2e-2
        a = _accf(acc[r * 5:r * 5 + t], shift)
        for tk in range(t):
            want = np.zeros(maxn)
            for p_, val in ra[tk].items():
                want[p_] = val
            assert np.abs(a[tk] - want).max() <= 2e-2
        if t < 5:
            assert acc[r * 5 + t:r * 5 + 5].abs().max().item() == 0  # rows of absent tokens untouched
        q0 += t


def test_topk_golden_kats(golden_topk):
    n = len([k for k in golden_topk if k.endswith(".values")])
    for dt in (torch.float64,):
        for i in range(n):
            v = torch.from_numpy(golden_topk[f"t{i}.values"]).to(DEV, dt)
            b = int(golden_topk[f"t{i}.budget"])
            take = min(b, v.numel())
            out = torch.empty(1, max(take, 1), dtype=torch.int32, device=DEV)
            ln = torch.empty(1, dtype=torch.int32, device=DEV)
            K.topk(v[None], torch.tensor([v.numel()], dtype=torch.int32, device=DEV),
                   torch.tensor([b], dtype=torch.int32, device=DEV), out, ln)
            assert int(ln.item()) == take
            assert out[0, :take].cpu().tolist() == golden_topk[f"t{i}.positions"].tolist()


def test_topk_random_float32_vs_stable_sort():
    rng = np.random.default_rng(11)
    for trial in range(300):
        n = int(rng.integers(1, 20000))
        v = rng.normal(size=n).astype(np.float32)
        if trial % 3 == 0:
            v = np.round(v, 1).astype(np.float32)
        if trial % 4 == 0:
            v = np.abs(v) * (rng.random(n) < 0.1)  # mostly exact zeros (planted-like ties)
        b = int(rng.integers(1, n + 2))
        want = O.topk_ascending(v.astype(np.float64), b)
        out = torch.empty(1, max(min(b, n), 1), dtype=torch.int32, device=DEV)
        ln = torch.empty(1, dtype=torch.int32, device=DEV)
        K.topk(torch.from_numpy(v).to(DEV)[None], torch.tensor([n], dtype=torch.int32, device=DEV),
               torch.tensor([b], dtype=torch.int32, device=DEV), out, ln)
        assert out[0, : min(b, n)].cpu().tolist() == want.tolist()


def test_select_critical_budget_and_rows(golden_budgets):
    rng = np.random.default_rng(3)
    B, rows, W = 6, 5, 9000
    shift = 40
    acc_h = rng.integers(0, 1 << 40, size=(B, rows, W), dtype=np.int64)
    acc_h[2] = 0  # all ties
    acc_h[4] = (acc_h[4] >> 36) << 36  # coarse values: many ties
    acc = torch.from_numpy(acc_h).to(DEV)
    kv_len = np.array([0, 1, 4000, 8999, 1000, 560], dtype=np.int32)
    n_rows = np.array([1, 2, 3, 5, 4, 1], dtype=np.int32)
    for s in (0.05, 0.07, 0.01, 1.0):
        imp = torch.zeros(B, W, dtype=torch.float64, device=DEV)
        crit = torch.zeros(B, W, dtype=torch.int32, device=DEV)
        clen = torch.zeros(B, dtype=torch.int32, device=DEV)
        bud = torch.zeros(B, dtype=torch.int32, device=DEV)
        K.select_critical(acc, acc.stride(0), acc.stride(1), shift, torch.from_numpy(n_rows).to(DEV),
                          torch.from_numpy(kv_len).to(DEV), s, B, imp, crit, clen, bud)
        torch.cuda.synchronize()
        for r in range(B):
            n = int(kv_len[r])
            got_imp = imp[r, :n].cpu().numpy()
            # fixed point -> fp64, rows ascending: exact (every partial sum < 2^53 units)
            want_imp = acc_h[r, : n_rows[r], :n].astype(np.float64).sum(axis=0) * 2.0 ** -shift
            assert np.array_equal(got_imp, want_imp)
            b = O.budget_for(n, s)
            assert int(bud[r]) == b
            want = O.topk_ascending(want_imp, b) if n else np.zeros(0, dtype=np.int64)
            assert int(clen[r]) == min(b, n)
            assert crit[r, : min(b, n)].cpu().tolist() == want.tolist()
    # device budget formula == reference on every golden (n, s)
    for n, s, b in golden_budgets:
        if n > W:
            continue
        clen = torch.zeros(1, dtype=torch.int32, device=DEV)
        bud = torch.zeros(1, dtype=torch.int32, device=DEV)
        K.select_critical(acc, 0, acc.stride(1), shift, torch.tensor([1], dtype=torch.int32, device=DEV),
                          torch.tensor([n], dtype=torch.int32, device=DEV), s, 1,
                          torch.zeros(1, W, dtype=torch.float64, device=DEV),
                          torch.zeros(1, W, dtype=torch.int32, device=DEV), clen, bud)
        assert int(bud.item()) == b, (n, s)


def test_argmax_and_accept():
    rng = np.random.default_rng(4)
    for dt in (torch.float32, torch.bfloat16, torch.float64):
        logits = rng.normal(size=(37, 151936)).astype(np.float32)
        logits[3, [5, 9, 100]] = 50.0  # tie -> lowest id
        logits[4, :] = 1.0
        t = torch.from_numpy(logits).to(DEV, dt)
        out = torch.empty(37, dtype=torch.int32, device=DEV)
        K.argmax_rows(t, out)
        want = np.argmax(t.double().cpu().numpy(), axis=1)
        assert out.cpu().numpy().tolist() == want.tolist()
    # fp64 rows whose top two differ below fp32 resolution: compared in fp64 (model.py:388-390)
    r64 = torch.zeros(2, 1000, dtype=torch.float64, device=DEV)
    r64[0, 10], r64[0, 900] = 1.0, 1.0 + 1e-12
    r64[1, 20], r64[1, 7] = 3.0, 3.0 - 1e-13
    out = torch.empty(2, dtype=torch.int32, device=DEV)
    K.argmax_rows(r64, out)
    assert out.cpu().tolist() == [900, 20]
    # accept rule (engine.py:231-239)
    targets = torch.tensor([5, 6, 7, 8, 9, 1, 2, 3, 4], dtype=torch.int32, device=DEV)
    tokens = torch.tensor([0, 5, 6, 0, 9, 0, 2, 9, 4], dtype=torch.int32, device=DEV)
    row0 = torch.tensor([0, 5, 8], dtype=torch.int32, device=DEV)
    nrows = torch.tensor([5, 3, 1], dtype=torch.int32, device=DEV)
    acc_, bonus = torch.empty(3, dtype=torch.int32, device=DEV), torch.empty(3, dtype=torch.int32, device=DEV)
    K.greedy_accept(targets, tokens, row0, nrows, acc_, bonus)
    assert acc_.cpu().tolist() == [2, 0, 0]
    assert bonus.cpu().tolist() == [7, 1, 4]


def test_rope_kv_write_matches_oracle():
    rng = np.random.default_rng(2)
    Hq, Hkv, d, L = 8, 2, 32, 2
    pool = _pool(L, Hkv, d, 300, 2, torch.float32)
    rows = 6
    qkv = torch.from_numpy(rng.normal(size=(rows, (Hq + 2 * Hkv) * d))).to(DEV, torch.float32)
    pos = np.array([0, 1, 17, 100, 255, 299], dtype=np.int32)
    tab = np.array([0, 1, 0, 1, 1, 0], dtype=np.int32)
    q_out = torch.empty(rows, Hq, d, dtype=torch.float32, device=DEV)
    K.rope_kv_write(qkv, torch.from_numpy(tab).to(DEV), torch.from_numpy(pos).to(DEV), pool, 1, Hq, q_out)
    torch.cuda.synchronize()
    x = qkv.double().cpu().numpy()
    for r in range(rows):
        want_q = O.rope(x[r, : Hq * d].reshape(Hq, d), int(pos[r]), d)
        want_k = O.rope(x[r, Hq * d:(Hq + Hkv) * d].reshape(Hkv, d), int(pos[r]), d)
        want_v = x[r, (Hq + Hkv) * d:].reshape(Hkv, d)
        kk, vv = pool.read(int(tab[r]), [int(pos[r])])
        assert np.abs(q_out[r].double().cpu().numpy() - want_q).max() < 1e-5
        assert np.abs(kk[0, 1].double().cpu().numpy() - want_k).max() < 1e-5
        assert np.array_equal(vv[0, 1].double().cpu().numpy(), want_v.astype(np.float32).astype(np.float64))


def _verify_case(n0s, nq, G, Hkv=8, seed=0, shuffle=5, scale=1.0, planted=(), page=16, lo=0):
    """One launch of len(n0s) verify items (nq tokens each) vs the oracle: outputs, lse and
    per-token fixed-point scores (model.py:229-253, selection.py:78-135).  ``lo``: the
    items' dense range starts there (a window; lo % 16 != 0 takes the cp.async producer)."""
    rng = np.random.default_rng(seed)
    d, Hq = 128, Hkv * G
    B = len(n0s)
    maxn = max(n0s) + nq
    pool = _pool(1, Hkv, d, maxn, B, torch.bfloat16, page=page, shuffle_seed=shuffle)
    for r, n in enumerate(n0s):
        _fill(pool, r, n + nq, rng, scale=scale)
    items = make_items([(r, r * nq, nq, n, 0, 0, lo, r * nq, 1) for r, n in enumerate(n0s)], DEV)
    q = torch.from_numpy(rng.normal(size=(B * nq, Hq, d))).to(DEV, torch.bfloat16)
    out = torch.empty_like(q)
    lse = torch.empty(B * nq, Hq, dtype=torch.float32, device=DEV)
    acc, shift = _acc(B * nq, maxn, Hq)
    K.attention(q, out, pool, 0, items, B, maxn, nq, Hq, lse=lse, acc=acc, acc_row_stride=maxn, acc_shift=shift,
                planted=torch.tensor(planted, dtype=torch.int32, device=DEV) if planted else None,
                planted_bonus=1.5 if planted else 0.0)
    torch.cuda.synchronize()
    for r, n in enumerate(n0s):
        kr, vr = pool.read(r, range(n + nq))
        kr, vr = kr.double().cpu().numpy()[:, 0], vr.double().cpu().numpy()[:, 0]
        sl = slice(r * nq, (r + 1) * nq)
        ro, rl, ra = _ref_rows(q[sl].double().cpu().numpy(), kr, vr, Hq, Hkv, d, [], range(lo, n + nq), n,
                               planted=planted, bonus=1.5)
        assert np.abs(out[sl].double().cpu().numpy() - ro).max() <= 2e-2, (r, n)
        assert np.abs(lse[sl].double().cpu().numpy() - rl).max() <= 2e-2, (r, n)
        a = _accf(acc[sl], shift)
        for t in range(nq):
            want = np.zeros(maxn)
            for p_, val in ra[t].items():
                want[p_] = val
            assert np.abs(a[t] - want).max() <= 2e-2, (r, n, t)
    return acc


@pytest.mark.parametrize("k", [2, 4, 8])
@pytest.mark.parametrize("G", [4, 8])
def test_verify_k_by_group_bf16(k, G):
    """configs[4]'s verify envelope: k+1 tokens x GQA group rows (12 .. 72 -> NR 16 .. 72)
    on the tcgen05 kernel, several items of different context in one launch."""
    _verify_case([4096, 1500, 129, 3], k + 1, G, seed=100 * k + G)


@pytest.mark.parametrize("G,n0", [(4, 20475), (4, 22000), (4, 1270), (8, 12283), (8, 13000), (4, 40000)])
def test_verify_tmem_slot_edges_bf16(G, n0):
    """Per-CTA tile counts at / just past the TMEM-resident slot count (the slot that doubles
    as the O accumulator is consumed first), below it, and far past it (evicted tiles
    recomputed)."""
    _verify_case([n0], 5, G, Hkv=2, seed=n0, scale=0.5)


def test_verify_single_token_bf16():
    """Greedy-decode shape: one query token (4 or 8 rows -> NR 8) over a dense context."""
    for G in (4, 8):
        _verify_case([3000, 700], 1, G, seed=G)


@pytest.mark.parametrize("G,rows", [(4, 48), (4, 64), (8, 48), (8, 80)])
def test_prefill_chunks_share_one_score_row_bf16(G, rows):
    """Prefill work items (BatchedDecoder._prefill_group): a 300-token prompt split into
    windows of rows/G tokens, every window summing its scores into ONE accumulator row
    (acc_step = 0, engine.py:192: all prompt rows count)."""
    rng = np.random.default_rng(rows + G)
    Hkv, d = 4, 128
    Hq = Hkv * G
    P = 300
    pool = _pool(1, Hkv, d, P, 1, torch.bfloat16, shuffle_seed=2)
    _fill(pool, 0, P, rng)
    kr, vr = pool.read(0, range(P))
    kr, vr = kr.double().cpu().numpy()[:, 0], vr.double().cpu().numpy()[:, 0]
    step = rows // G
    items = make_items([(0, q0, min(step, P - q0), q0, 0, 0, 0, 0, 0) for q0 in range(0, P, step)], DEV)
    n_items = -(-P // step)
    q = torch.from_numpy(rng.normal(size=(P, Hq, d))).to(DEV, torch.bfloat16)
    out = torch.empty_like(q)
    shift = K.score_shift(P, 1, Hq)
    acc = torch.zeros(1, P, dtype=torch.int64, device=DEV)
    K.attention(q, out, pool, 0, items, n_items, P, step, Hq, acc=acc, acc_row_stride=P, acc_shift=shift)
    torch.cuda.synchronize()
    ro, _, ra = _ref_rows(q.double().cpu().numpy(), kr, vr, Hq, Hkv, d, [], range(P), 0)
    assert np.abs(out.double().cpu().numpy() - ro).max() <= 2e-2
    want = np.zeros(P)
    for t in range(P):
        for p_, val in ra[t].items():
            want[p_] += val
    got = _accf(acc, shift)[0]
    np.testing.assert_allclose(got.sum(), P * Hq, rtol=1e-2)
    assert np.abs(got - want).max() <= 2e-2 * max(1.0, want.max())


def test_score_accumulation_is_bitwise_deterministic_bf16():
    """The fixed-point score reductions land in any order across heads and cluster CTAs;
    the accumulated integers must not depend on it (repeat launches, bitwise)."""
    rng = np.random.default_rng(9)
    Hkv, G, d, nq = 8, 4, 128, 5
    Hq = Hkv * G
    lens = [6000, 3000, 8000, 100]
    maxn = max(lens) + nq
    pool = _pool(1, Hkv, d, maxn, len(lens), torch.bfloat16, shuffle_seed=3)
    for r, n in enumerate(lens):
        _fill(pool, r, n + nq, rng)
    items = make_items([(r, r * nq, nq, n, 0, 0, 0, r * nq, 1) for r, n in enumerate(lens)], DEV)
    q = torch.from_numpy(rng.normal(size=(len(lens) * nq, Hq, d))).to(DEV, torch.bfloat16)
    out = torch.empty_like(q)
    runs = []
    for _ in range(4):
        acc, shift = _acc(len(lens) * nq, maxn, Hq, L=36)
        for layer_rep in range(3):  # several "layers" accumulate into the same rows
            K.attention(q, out, pool, 0, items, len(lens), maxn, nq, Hq, acc=acc, acc_row_stride=maxn,
                        acc_shift=shift)
        runs.append(acc.cpu())
    for r in runs[1:]:
        assert torch.equal(r, runs[0])


def test_rope_kv_write_bf16_matches_oracle():
    """K5 bf16 branch: rotated q / k rounded to bf16 once, v copied exactly (model.py:212-222)."""
    rng = np.random.default_rng(12)
    Hq, Hkv, d, L = 16, 4, 128, 2
    pool = _pool(L, Hkv, d, 9000, 2, torch.bfloat16)
    rows = 7
    qkv = torch.from_numpy(rng.normal(size=(rows, (Hq + 2 * Hkv) * d))).to(DEV, torch.bfloat16)
    pos = np.array([0, 1, 17, 100, 4095, 8191, 8999], dtype=np.int32)
    tab = np.array([0, 1, 0, 1, 1, 0, 1], dtype=np.int32)
    q_out = torch.empty(rows, Hq, d, dtype=torch.bfloat16, device=DEV)
    K.rope_kv_write(qkv, torch.from_numpy(tab).to(DEV), torch.from_numpy(pos).to(DEV), pool, 1, Hq, q_out)
    torch.cuda.synchronize()
    x = qkv.double().cpu().numpy()
    for r in range(rows):
        want_q = O.rope(x[r, : Hq * d].reshape(Hq, d), int(pos[r]), d)
        want_k = O.rope(x[r, Hq * d:(Hq + Hkv) * d].reshape(Hkv, d), int(pos[r]), d)
        want_v = x[r, (Hq + Hkv) * d:].reshape(Hkv, d)
        kk, vv = pool.read(int(tab[r]), [int(pos[r])])
        # one bf16 rounding of the fp32 rotation: |err| <= 2^-8 |x| + fp32 angle error at 9K positions
        assert np.abs(q_out[r].double().cpu().numpy() - want_q).max() <= 1e-2 * max(1.0, np.abs(want_q).max())
        assert np.abs(kk[0, 1].double().cpu().numpy() - want_k).max() <= 1e-2 * max(1.0, np.abs(want_k).max())
        assert np.array_equal(vv[0, 1].double().cpu().numpy(), want_v)


@pytest.mark.parametrize("R", [1, 37, 228])
@pytest.mark.parametrize("N,Kd", [(512, 256), (4096, 4096), (8192, 4096)])
def test_linear_tuned_cublaslt_matches_fp32(R, N, Kd):
    """sd_linear (the tuned cuBLASLt path of the layer loop and the LM head, model.py:326-339)
    vs a torch fp32 matmul of the same bf16 inputs: bf16 / fp32 outputs, overwrite / accumulate."""
    g = torch.Generator(device=DEV)
    g.manual_seed(R + N + Kd)
    a = (torch.randn(R, Kd, device=DEV, generator=g) * 0.5).to(torch.bfloat16)
    w = (torch.randn(N, Kd, device=DEV, generator=g) * 0.05).to(torch.bfloat16)
    ref = a.float() @ w.float().t()
    out = torch.empty(R, N, dtype=torch.float32, device=DEV)
    K.linear(a, w, out)
    x0 = torch.randn(R, N, device=DEV, generator=g)
    x = x0.clone()
    K.linear(a, w, x, accumulate=True)
    ob = torch.empty(R, N, dtype=torch.bfloat16, device=DEV)
    K.linear(a, w, ob)
    torch.cuda.synchronize()
    scale = ref.abs().max().item()
    assert (out - ref).abs().max().item() <= 1e-3 * scale + 1e-4
    assert (x - (x0 + ref)).abs().max().item() <= 1e-3 * scale + 1e-4
    assert (ob.float() - ref).abs().max().item() <= 1e-2 * scale + 1e-3


@pytest.mark.parametrize("G", [4, 8])
def test_fused_verify_draft_launch_matches_separate_launches(G):
    """f3: verify items (dense, score emission) and draft items (critical list + fresh tail) in
    ONE launch (sd_attention_pair) give bitwise the outputs and fixed-point scores of the two
    separate launches (same tcgen05 bodies), and the separate launches match the oracle
    (tests above)."""
    rng = np.random.default_rng(50 + G)
    Hkv, d, nq = 8, 128, 5
    Hq = Hkv * G
    lens_v = [4000, 1200, 2600]
    lens_d = [3000, 800, 5000, 1700, 2200]
    B = len(lens_v) + len(lens_d)
    maxn = max(lens_v + lens_d) + nq
    pool = _pool(1, Hkv, d, maxn, B, torch.bfloat16, shuffle_seed=7)
    for r, n in enumerate(lens_v + lens_d):
        _fill(pool, r, n + nq, rng, scale=0.5)
    nv = len(lens_v)
    v_items = make_items([(r, r * nq, nq, n, 0, 0, 0, r * nq, 1) for r, n in enumerate(lens_v)], DEV)
    bud = [max(1, n // (20 if G == 4 else 40)) for n in lens_d]  # critical lists stay TMEM-resident
    crit = np.zeros((len(lens_d), max(bud)), dtype=np.int32)
    for i, n in enumerate(lens_d):
        crit[i, :bud[i]] = np.sort(rng.choice(n, bud[i], replace=False))
    crit_d = torch.from_numpy(crit.reshape(-1)).to(DEV)
    j = 2  # third draft of the round: fresh tail n .. n + 2
    d_rows = [(nv + i, nv * nq + i, 1, n + j, i * crit.shape[1], bud[i], n, -1, 0) for i, n in enumerate(lens_d)]
    d_items = make_items(d_rows, DEV)
    R = nv * nq + len(lens_d)
    q = torch.from_numpy(rng.normal(size=(R, Hq, d))).to(DEV, torch.bfloat16)
    runs = []
    for fused in (False, True):
        out = torch.zeros(R, Hq, d, dtype=torch.bfloat16, device=DEV)
        acc, shift = _acc(nv * nq, maxn, Hq)
        v = dict(items=v_items, num_items=nv, max_keys=maxn, max_nq=nq, acc=acc, acc_row_stride=maxn, acc_shift=shift)
        dr = dict(items=d_items, num_items=len(lens_d), max_keys=max(bud) + j + 1, crit=crit_d)
        if fused:
            assert K.attention_pair(q, out, pool, 0, v, dr, Hq)
        else:
            K.attention(q, out, pool, 0, v_items, nv, maxn, nq, Hq, acc=acc, acc_row_stride=maxn, acc_shift=shift)
            K.attention(q, out, pool, 0, d_items, len(lens_d), max(bud) + j + 1, 1, Hq, crit=crit_d)
        torch.cuda.synchronize()
        runs.append((out.clone(), acc.clone()))
    assert torch.equal(runs[0][0], runs[1][0])
    assert torch.equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("page,lo", [(32, 0), (64, 0), (16, 37), (16, 512)])
def test_verify_page_sizes_and_windows_bf16(page, lo):
    """K2 producer paths: TMA 16-key boxes inside 32 / 64-token pages, a window starting off a
    16-key boundary (cp.async rows) and on one (TMA)."""
    _verify_case([3000, 1100, 4500], 5, 4, seed=page + lo, page=page, lo=lo)
