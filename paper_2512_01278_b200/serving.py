"""Batched unified draft/verify execution on one B200.

``BatchedDecoder`` runs one iteration of the unified scheduler as ONE batched
forward: every draft member contributes 1 row (K1 work item over its critical
set + fresh tail), every verify member round_target+1 rows (K2 work item over
its whole context with score emission), weights are read once per iteration
(PAPER.md:443-453), then K4 (argmax + accept) and K3 (critical refresh) run
for the verify members.  Host state per request mirrors engine.RequestState.

``run_token_sim`` is the drop-in for the reference's token-level serving loop
(simulate.py:271-548): admission in arrival order, PhaseBuckets placement,
KvPool page accounting, form_batch / step_pipeline, free_tail rollback —
with the per-member engine calls replaced by one BatchedDecoder.step().
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import kernels as K
from .engine import DecodeRequest, RoundRecord, RoundStats
from .errors import ConfigurationError, ContractError, SimulationError
from .model import AttnLaunch, ToyModel, forward_rows, lm_head
from .paged import PagedKvPool
from .selection import compute_budget

# rows per prefill work item (query tokens x GQA group); the tcgen05 verify kernel takes up to
# 80 rows, two CTAs per SM up to 48
MMA_MAX_ROWS = int(os.environ.get("SD_PREFILL_ROWS", "48"))


@dataclass
class Seq:
    """Host state of one request inside the batched decoder."""

    request_id: int
    slot: int
    prompt: list
    max_output: int
    eos_token: int | None
    k: int
    committed: list = field(default_factory=list)
    drafted: list = field(default_factory=list)
    phase: int = 0
    round_target: int = 0
    n_kv: int = 0            # committed KV rows (prompt + committed - 1)
    crit_len: int = 0
    budget: int = 0
    done: bool = False
    stats: RoundStats | None = None

    @property
    def kv_len(self) -> int:
        return len(self.prompt) + len(self.committed) + len(self.drafted)


@dataclass
class StepResult:
    accepted: dict
    emitted: int
    rows: int
    draft_rows: int
    verify_rows: int


class BatchedDecoder:
    def __init__(self, model: ToyModel, k: int, sparsity: float, max_requests: int, max_seq_len: int,
                 page_size: int = 16, pool_tokens: int | None = None):
        if k < 1:
            raise ConfigurationError("k must be at least 1")
        if not 0.0 < sparsity <= 1.0:
            raise ConfigurationError("sparsity must lie in (0, 1]")
        c = model.config
        self.model, self.k, self.sparsity = model, k, sparsity
        self.dev = model.device
        self.max_requests = max_requests
        self.max_seq_len = max_seq_len + k + 1
        pages_per_row = -(-self.max_seq_len // page_size)
        pool_pages = pages_per_row * max_requests if pool_tokens is None else -(-pool_tokens // page_size)
        self.pool = PagedKvPool(c.num_layers, c.num_kv_heads, c.head_dim, pool_pages, page_size, max_requests,
                                pages_per_row, model.dtype, self.dev)
        self.crit_cap = max(1, compute_budget(self.max_seq_len, sparsity))
        self.crit = torch.zeros(max_requests, self.crit_cap, dtype=torch.int32, device=self.dev)
        self.crit_len_dev = torch.zeros(max_requests, dtype=torch.int32, device=self.dev)
        self.acc_w = self.max_seq_len
        # fixed-point score accumulators (kernels.score_shift): one row per verify query token
        self.acc = torch.zeros(max_requests * (k + 1), self.acc_w, dtype=torch.int64, device=self.dev)
        self.imp = torch.zeros(max_requests, self.acc_w, dtype=torch.float64, device=self.dev)
        self.verify_shift = K.score_shift(1, c.num_layers, c.num_q_heads)
        self.prefill_shift = K.score_shift(self.max_seq_len, c.num_layers, c.num_q_heads)  # prompt rows sum
        self.free_slots = list(range(max_requests - 1, -1, -1))
        self.seqs: dict = {}
        self._host_kv: dict = {}     # request -> {position: (K rows, V rows)} pinned host copies
        self.offloaded_bytes = 0
        self.reloaded_bytes = 0
        self.attn_timer = None       # optional callable(kind, start) for per-launch timing
        self.host_times: list = []   # per step: (host enqueue s, enqueue + device drain s)
        self.last_rows = 0

    # -- lifecycle ------------------------------------------------------------------
    def _alloc_slot(self, req: DecodeRequest) -> Seq:
        if not self.free_slots:
            raise ContractError("no free request slot in the batched decoder")
        if not req.prompt:
            raise ContractError("prompt must be non-empty")
        if req.max_output < 1:
            raise ConfigurationError("max_output must be at least 1")
        need = len(req.prompt) + req.max_output + self.k + 1
        if need > self.max_seq_len:
            raise ContractError(f"request needs {need} KV positions > decoder max {self.max_seq_len}")
        slot = self.free_slots.pop()
        self.pool.ensure_tokens(slot, need)
        s = Seq(request_id=req.request_id, slot=slot, prompt=list(req.prompt), max_output=req.max_output,
                eos_token=req.eos_token, k=self.k, round_target=self.k, stats=RoundStats(k=self.k))
        self.seqs[req.request_id] = s
        return s

    def release(self, request_id) -> None:
        s = self.seqs.pop(request_id)
        self.pool.release_row(s.slot)
        self.free_slots.append(s.slot)
        self._host_kv.pop(request_id, None)

    # -- host offload tier (kvpool.py:213-237,272-311) -----------------
    def offload_positions(self, request_id, positions) -> int:
        """Copy the K/V rows of ``positions`` (all layers) to pinned host memory and return
        every physical page whose tokens are all on the host to the device pool.  The
        request must not be scheduled until ``reload_positions`` brings them back."""
        positions = sorted(int(p) for p in positions)
        s = self.seqs.get(request_id)
        if s is None or not positions:
            return 0
        k, v = self.pool.read(s.slot, positions)  # (n, L, Hkv, d)
        hk = torch.empty(k.shape, dtype=k.dtype, pin_memory=True)
        hv = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
        hk.copy_(k, non_blocking=True)
        hv.copy_(v, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        store = self._host_kv.setdefault(request_id, {})
        for i, p in enumerate(positions):
            store[p] = (hk[i], hv[i])
        ps = self.pool.page_size
        whole = sorted({p // ps for p in positions if all(q in store for q in range(p // ps * ps, p // ps * ps + ps))})
        self.pool.unmap_pages(s.slot, whole)
        self.offloaded_bytes += 2 * k.numel() * k.element_size()
        return len(positions)

    def reload_positions(self, request_id, positions) -> int:
        """Inverse of ``offload_positions``: remap pages and copy the rows back."""
        positions = sorted(int(p) for p in positions)
        s = self.seqs.get(request_id)
        store = self._host_kv.get(request_id)
        if s is None or not positions or store is None:
            return 0
        ps = self.pool.page_size
        self.pool.remap_pages(s.slot, sorted({p // ps for p in positions}))
        self.pool.sync_table()
        # a remapped page receives every row it holds: also the still-host rows of pages
        # that were only partly reloaded stay on the host and are written when they return
        k = torch.stack([store[p][0] for p in positions])
        v = torch.stack([store[p][1] for p in positions])
        self.pool.write(s.slot, positions, k, v)
        for p in positions:
            del store[p]
        self.reloaded_bytes += 2 * k.numel() * k.element_size()
        return len(positions)

    def _emit(self, s: Seq, toks) -> int:
        landed = 0
        for t in toks:
            if len(s.committed) >= s.max_output:
                break
            s.committed.append(int(t))
            landed += 1
            if s.eos_token is not None and int(t) == s.eos_token:
                s.done = True
                break
        if len(s.committed) >= s.max_output:
            s.done = True
        return landed

    # -- prefill ------------------------------------------------------------------------
    def prefill(self, requests, max_rows: int = 32768) -> list:
        """Prompt pass with score capture for a group of new requests.  Seeds
        the first critical set from all prompt rows (engine.py:154-193)."""
        seqs = [self._alloc_slot(r) for r in requests]
        self.pool.sync_table()
        group: list = []
        rows = 0
        for s in seqs:
            if group and rows + len(s.prompt) > max_rows:
                self._prefill_group(group)
                group, rows = [], 0
            group.append(s)
            rows += len(s.prompt)
        if group:
            self._prefill_group(group)
        return seqs

    def prefill_synthetic(self, requests, real_tokens: int, max_rows: int = 32768, seed: int = 0) -> list:
        """Benchmark setup: the model prefill (scores captured) runs on the first
        ``real_tokens`` of each prompt; the K/V rows of the remaining prompt positions (a
        teacher-forced continuation) are written directly as synthetic N(0, 1) values,
        which changes no kernel's work, and the first critical set is re-selected over
        the full length from the real prefix's scores."""
        full = [list(r.prompt) for r in requests]
        short = [DecodeRequest(r.request_id, list(r.prompt[:real_tokens]), r.max_output, r.eos_token)
                 for r in requests]
        seqs = [self._alloc_slot(r) for r in requests]  # capacity for the full length
        for s, r in zip(seqs, short):
            s.prompt = list(r.prompt)
        self.pool.sync_table()
        group, rows = [], 0
        for s in seqs:
            if group and rows + len(s.prompt) > max_rows:
                self._prefill_group(group)
                group, rows = [], 0
            group.append(s)
            rows += len(s.prompt)
        if group:
            self._prefill_group(group)
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        c = self.model.config
        refresh = []
        for s, pr in zip(seqs, full):
            extra = list(range(len(s.prompt), len(pr)))
            if extra:
                slots = self.pool.slots(s.slot, extra).to(self.dev)
                shape = (c.num_layers, len(extra), c.num_kv_heads, c.head_dim)
                self.pool.k[:, slots] = torch.randn(shape, generator=g, device=self.dev).to(self.pool.dtype)
                self.pool.v[:, slots] = torch.randn(shape, generator=g, device=self.dev).to(self.pool.dtype)
            s.prompt = pr
            s.n_kv = len(pr)
            if not s.done:
                refresh.append((s, 1))
        self._refresh(refresh, self.prefill_shift)
        return seqs

    def _prefill_group(self, seqs) -> None:
        c = self.model.config
        G = c.group_size
        chunk = max(1, MMA_MAX_ROWS // G)
        toks, rt, rp, items = [], [], [], []
        row = 0
        for s in seqs:
            P = len(s.prompt)
            toks.extend(s.prompt)
            rt.extend([s.slot] * P)
            rp.extend(range(P))
            acc_row = s.slot * (self.k + 1)
            for q0 in range(0, P, chunk):
                nq = min(chunk, P - q0)
                items.append((s.slot, row + q0, nq, q0, 0, 0, 0, acc_row, 0))
            row += P
        max_p = max(len(s.prompt) for s in seqs)
        self.acc.view(self.max_requests, self.k + 1, self.acc_w)[[s.slot for s in seqs], 0] = 0
        shift = self.prefill_shift  # all prompt rows sum into one accumulator row
        tok = torch.tensor(toks, dtype=torch.int32, device=self.dev)
        launch = AttnLaunch(_items(items, self.dev), len(items), max_p, min(chunk, max_p), acc=self.acc,
                            acc_row_stride=self.acc_w, acc_shift=shift)
        x = forward_rows(self.model, self.pool, tok, _i32(rt, self.dev), _i32(rp, self.dev), [launch])
        last = torch.tensor(np.cumsum([len(s.prompt) for s in seqs]) - 1, device=self.dev)
        first = _argmax(lm_head(self.model, x.index_select(0, last))).cpu().tolist()
        refresh = []
        for s, t in zip(seqs, first):
            s.n_kv = len(s.prompt)
            s.stats.full_forwards += 1
            self._emit(s, [t])
            s.stats.emitted_tokens = len(s.committed)
            if not s.done:
                refresh.append((s, 1))
        self._refresh(refresh, shift)

    def _refresh(self, pairs, shift: int) -> None:
        """K3 for (seq, surviving rows) pairs: importance -> budget -> top-k."""
        if not pairs:
            return
        slots = [s.slot for s, _ in pairs]
        n_rows = [n for _, n in pairs]
        kv = [s.n_kv for s, _ in pairs]
        K.select_critical(self.acc, (self.k + 1) * self.acc.stride(0), self.acc.stride(0), shift, _i32(n_rows, self.dev),
                          _i32(kv, self.dev), self.sparsity, len(pairs), self.imp, self.crit, self.crit_len_dev,
                          req_index=_i32(slots, self.dev))
        for s, _ in pairs:
            s.budget = compute_budget(s.n_kv, self.sparsity)
            s.crit_len = min(s.budget, s.n_kv)

    # -- one unified iteration --------------------------------------------------------------
    def step(self, draft_ids, verify_ids) -> StepResult:
        """Run every draft member one draft step and every verify member its
        verification, as one batched forward (engine.py:196-260 semantics)."""
        c = self.model.config
        t_host0 = time.perf_counter()
        toks, rt, rp = [], [], []
        d_items, v_items = [], []
        drafts = [self.seqs[r] for r in draft_ids]
        verifs = [self.seqs[r] for r in verify_ids]
        row = 0
        d_max_keys = 1
        for s in drafts:
            if s.done or s.phase >= s.round_target:
                raise ContractError(f"request {s.request_id} cannot draft now")
            tok = s.drafted[-1] if s.drafted else s.committed[-1]
            pos = s.n_kv + s.phase
            toks.append(tok)
            rt.append(s.slot)
            rp.append(pos)
            d_items.append((s.slot, row, 1, pos, s.slot * self.crit_cap, s.crit_len, s.n_kv, -1, 0))
            d_max_keys = max(d_max_keys, s.crit_len + s.phase + 1)
            row += 1
        n_draft_rows = row
        v_row0, v_n = [], []
        v_max_keys, v_max_nq = 1, 1
        for s in verifs:
            if s.done or s.phase != s.round_target:
                raise ContractError(f"request {s.request_id} cannot verify now")
            seq_toks = [s.committed[-1], *s.drafted]
            t = len(seq_toks)
            toks.extend(seq_toks)
            rt.extend([s.slot] * t)
            rp.extend(range(s.n_kv, s.n_kv + t))
            v_items.append((s.slot, row, t, s.n_kv, 0, 0, 0, s.slot * (self.k + 1), 1))
            v_row0.append(row)
            v_n.append(t)
            v_max_keys = max(v_max_keys, s.n_kv + t)
            v_max_nq = max(v_max_nq, t)
            row += t
        R = row
        if R == 0:
            return StepResult({}, 0, 0, 0, 0)
        launches = []
        if v_items:
            slots = torch.tensor([s.slot for s in verifs], device=self.dev)
            self.acc.view(self.max_requests, self.k + 1, self.acc_w)[slots] = 0
            launches.append(AttnLaunch(_items(v_items, self.dev), len(v_items), v_max_keys, v_max_nq, acc=self.acc,
                                       acc_row_stride=self.acc_w, acc_shift=self.verify_shift,
                                       timer=self._timer("verify")))
        if d_items:  # after the verify launch: it runs on the side stream (model.forward_rows)
            launches.append(AttnLaunch(_items(d_items, self.dev), len(d_items), d_max_keys, 1, crit=self.crit,
                                       timer=self._timer("draft")))
        tok_dev = _i32(toks, self.dev)
        x = forward_rows(self.model, self.pool, tok_dev, _i32(rt, self.dev), _i32(rp, self.dev), launches)
        targets = _argmax(lm_head(self.model, x))
        t_launched = time.perf_counter()
        if verifs:
            row0_d, n_d = _i32(v_row0, self.dev), _i32(v_n, self.dev)
            acc_d = torch.empty(len(verifs), dtype=torch.int32, device=self.dev)
            bonus_d = torch.empty_like(acc_d)
            K.greedy_accept(targets, tok_dev, row0_d, n_d, acc_d, bonus_d)
            host = torch.cat([targets, acc_d, bonus_d]).cpu().numpy()
        else:
            host = targets.cpu().numpy()
        t_synced = time.perf_counter()
        self.host_times.append((t_launched - t_host0, t_synced - t_host0))
        tg = host[:R]
        emitted = 0
        for i, s in enumerate(drafts):
            s.drafted.append(int(tg[i]))
            s.phase += 1
            s.stats.sparse_forwards += 1
        accepted = {}
        refresh = []
        for m, s in enumerate(verifs):
            a = int(host[R + m])
            bonus = int(host[R + len(verifs) + m])
            kv_at = s.kv_len
            drafts_m = s.drafted
            s.n_kv += a + 1  # KV rollback: rows beyond n_kv + a are dead
            landed = self._emit(s, drafts_m[:a] + [bonus])
            emitted += landed
            s.stats.emitted_tokens += landed
            s.stats.full_forwards += 1
            s.stats.rounds.append(RoundRecord(len(s.stats.rounds), len(drafts_m), a, kv_at, s.budget))
            s.drafted, s.phase, s.round_target = [], 0, self.k
            accepted[s.request_id] = a
            if not s.done:
                refresh.append((s, a + 1))
        self._refresh(refresh, self.verify_shift)
        self.last_rows = R
        return StepResult(accepted, emitted, R, n_draft_rows, R - n_draft_rows)

    def _timer(self, kind):
        if self.attn_timer is None:
            return None
        return lambda start: self.attn_timer(kind, start)


def _i32(vals, dev) -> torch.Tensor:
    return torch.from_numpy(np.asarray(vals, dtype=np.int32)).to(dev, non_blocking=True)


def _items(rows, dev) -> torch.Tensor:
    arr = np.zeros((max(1, len(rows)), N.ITEM_FIELDS), dtype=np.int32)
    if rows:
        arr[: len(rows), :9] = np.asarray(rows, dtype=np.int32)
    return torch.from_numpy(arr).to(dev, non_blocking=True)


def _argmax(logits: torch.Tensor) -> torch.Tensor:
    out = torch.empty(logits.shape[0], dtype=torch.int32, device=logits.device)
    K.argmax_rows(logits.contiguous(), out)
    return out
