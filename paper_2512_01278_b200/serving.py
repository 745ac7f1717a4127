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
    inflight: bool = False   # a submitted verification whose outcome the host has not applied
    n_kv_ub: int = 0         # upper bound of n_kv while inflight

    @property
    def kv_len(self) -> int:
        return len(self.prompt) + len(self.committed) + len(self.drafted)


@dataclass
class PendingStep:
    """A submitted iteration (BatchedDecoder.submit) awaiting BatchedDecoder.complete."""

    index: int
    ring: int
    verifs: list     # (seq, drafted count, kv_len at verify, budget of the round's set)
    drafts: list
    rows: int
    draft_rows: int
    event: object
    t_host0: float
    t_launched: float


@dataclass
class StepResult:
    accepted: dict
    emitted: int
    rows: int
    draft_rows: int
    verify_rows: int


class BatchedDecoder:
    def __init__(self, model: ToyModel, k: int, sparsity: float, max_requests: int, max_seq_len: int,
                 page_size: int = 16, pool_tokens: int | None = None, paging: str = "reserve"):
        """``paging``: "reserve" maps a request's whole lifetime (prompt + max_output + k + 1
        positions) at admission; "on_demand" maps physical pages as positions are written
        (prompt at admission, then each iteration's draft / verify rows), so a pool of
        ``pool_tokens`` holds as many requests as their CURRENT lengths allow — the physical
        side of KvPool's page accounting (kvpool.py:174-237)."""
        if paging not in ("reserve", "on_demand"):
            raise ConfigurationError("paging must be 'reserve' or 'on_demand'")
        self.on_demand = paging == "on_demand"
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
        # device-resident request state (csrc/pipeline.cu): the iteration's inputs are built and
        # its accept/rollback applied on the device, so the host can enqueue iteration i+1
        # before it reads iteration i's results (delayed verification processing)
        self.n_kv_dev = torch.zeros(max_requests, dtype=torch.int32, device=self.dev)
        self.last_tok_dev = torch.zeros(max_requests, dtype=torch.int32, device=self.dev)
        self.drafted_dev = torch.zeros(max_requests, k, dtype=torch.int32, device=self.dev)
        max_rows = max_requests * (k + 1)
        self._tok_buf = torch.zeros(max_rows, dtype=torch.int32, device=self.dev)
        self._rt_buf = torch.zeros(max_rows, dtype=torch.int32, device=self.dev)
        self._rp_buf = torch.zeros(max_rows, dtype=torch.int32, device=self.dev)
        self._targets = torch.zeros(max_rows, dtype=torch.int32, device=self.dev)
        self._v_items = torch.zeros(max_requests, N.ITEM_FIELDS, dtype=torch.int32, device=self.dev)
        self._d_items = torch.zeros(max_requests, N.ITEM_FIELDS, dtype=torch.int32, device=self.dev)
        self._sel = torch.zeros(3, max_requests, dtype=torch.int32, device=self.dev)
        self._res_dev = torch.zeros(max_requests, k + 2, dtype=torch.int32, device=self.dev)
        self._plan_dev = torch.zeros(max_requests, N.PLAN_FIELDS, dtype=torch.int32, device=self.dev)
        # pinned host rings: a plan buffer may be rewritten only after its H2D copy ran, a
        # result buffer is read after its D2H copy's event
        self._ring = 3
        self._plan_host = [torch.zeros(max_requests, N.PLAN_FIELDS, dtype=torch.int32, pin_memory=True)
                           for _ in range(self._ring)]
        self._res_host = [torch.zeros(max_requests, k + 2, dtype=torch.int32, pin_memory=True)
                          for _ in range(self._ring)]
        self._ring_ev = [None] * self._ring
        self._iter = 0
        self.free_slots = list(range(max_requests - 1, -1, -1))
        self.seqs: dict = {}
        self._host_kv: dict = {}     # request -> {position: (K rows, V rows)} pinned host copies
        self.offloaded_bytes = 0
        self.reloaded_bytes = 0
        self.attn_timer = None       # optional callable(kind, start) for per-launch timing (torch loop)
        self.attn_events = False     # record (start, end) events around every K1 / K2 launch
        self.keep_logits = False     # keep the last step's logits (diagnostics)
        self.last_logits = None
        self.last_events: dict = {}  # kind -> [(start, end)] per layer of the last submitted step
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
        slot = self.free_slots[-1]
        self.pool.ensure_tokens(slot, len(req.prompt) if self.on_demand else need)
        self.free_slots.pop()
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
    def _copy_stream(self) -> torch.cuda.Stream:
        st = getattr(self, "_copy_st", None)
        if st is None:
            st = self._copy_st = torch.cuda.Stream(self.dev)
        return st

    def offload_positions(self, request_id, positions) -> int:
        """Copy the K/V rows of ``positions`` (all layers) to pinned host memory on the copy
        stream and return every physical page whose tokens are all on the host to the
        device pool once that copy has completed (event-fenced, kvpool.py:213-237).  The
        request must not be scheduled until ``reload_positions`` brings them back."""
        positions = sorted(int(p) for p in positions)
        s = self.seqs.get(request_id)
        if s is None or not positions:
            return 0
        main = torch.cuda.current_stream(self.dev)
        cs = self._copy_stream()
        cs.wait_stream(main)                    # the rows were written by earlier compute
        slots = self.pool.slots(s.slot, positions)
        hk = torch.empty((len(positions), *self.pool.k.shape[:1], *self.pool.k.shape[2:]), dtype=self.pool.dtype,
                         pin_memory=True)
        hv = torch.empty_like(hk, pin_memory=True)
        with torch.cuda.stream(cs):
            sl = slots.to(self.dev, non_blocking=True)
            hk.copy_(self.pool.k[:, sl].transpose(0, 1), non_blocking=True)
            hv.copy_(self.pool.v[:, sl].transpose(0, 1), non_blocking=True)
            done = torch.cuda.Event()
            done.record(cs)
        store = self._host_kv.setdefault(request_id, {})
        for i, p in enumerate(positions):
            store[p] = (hk[i], hv[i], done)
        ps = self.pool.page_size
        whole = sorted({p // ps for p in positions if all(q in store for q in range(p // ps * ps, p // ps * ps + ps))})
        self.pool.unmap_pages(s.slot, whole, after=done)
        self.offloaded_bytes += 2 * hk.numel() * hk.element_size()
        return len(positions)

    def reload_positions(self, request_id, positions) -> int:
        """Inverse of ``offload_positions``: remap pages and copy the rows back on the copy
        stream; the compute stream waits for that copy before its next launch."""
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
        n = len(positions)
        hk = torch.empty((n, *store[positions[0]][0].shape), dtype=self.pool.dtype, pin_memory=True)
        hv = torch.empty_like(hk, pin_memory=True)
        for i, p in enumerate(positions):
            store[p][2].synchronize()           # its offload copy landed in host memory
            hk[i].copy_(store[p][0])
            hv[i].copy_(store[p][1])
            del store[p]
        if not store:
            del self._host_kv[request_id]
        main = torch.cuda.current_stream(self.dev)
        cs = self._copy_stream()
        cs.wait_stream(main)                    # fresh pages may have been freed by compute
        slots = self.pool.slots(s.slot, positions)
        with torch.cuda.stream(cs):
            sl = slots.to(self.dev, non_blocking=True)
            dk = hk.to(self.dev, non_blocking=True)
            dv = hv.to(self.dev, non_blocking=True)
            self.pool.k[:, sl] = dk.transpose(0, 1)
            self.pool.v[:, sl] = dv.transpose(0, 1)
        main.wait_stream(cs)
        self.reloaded_bytes += 2 * hk.numel() * hk.element_size()
        return n

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
        self.n_kv_dev.index_copy_(0, _i32([s.slot for s in seqs], self.dev).long(),
                                  _i32([s.n_kv for s in seqs], self.dev))
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
        first_dev = _argmax(lm_head(self.model, x.index_select(0, last)))
        slots_dev = _i32([s.slot for s in seqs], self.dev).long()
        self.last_tok_dev.index_copy_(0, slots_dev, first_dev)
        self.n_kv_dev.index_copy_(0, slots_dev, _i32([len(s.prompt) for s in seqs], self.dev))
        first = first_dev.cpu().tolist()
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
        verification, as one batched forward (engine.py:196-260 semantics), and
        process the results before returning (synchronous pipeline)."""
        return self.complete(self.submit(draft_ids, verify_ids))

    def submit(self, draft_ids, verify_ids) -> "PendingStep":
        """Enqueue one unified iteration without waiting for any device result.

        Input tokens, positions and work items come from the device-resident request
        state (sd_step_prepare); accept / rollback / critical refresh run on the device
        (sd_step_commit, K3).  The host mirrors only what scheduling needs: draft
        phases advance here, verify outcomes (accepted count, bonus, emitted tokens,
        done) arrive with ``complete`` — typically called for iteration i after
        iteration i+1 has been submitted (delayed verification processing,
        scheduler.py:135-197), which keeps the GPU busy while the host works."""
        c = self.model.config
        t_host0 = time.perf_counter()
        drafts = [self.seqs[r] for r in draft_ids]
        verifs = [self.seqs[r] for r in verify_ids]
        n_members = len(drafts) + len(verifs)
        j = self._iter % self._ring
        self._iter += 1
        if self._ring_ev[j] is not None:
            self._ring_ev[j].synchronize()   # its plan copy and result copy are done
        for s in drafts + verifs:
            if self.pool.has_unmapped(s.slot) or self._host_kv.get(s.request_id):
                # its block table points offloaded pages at a placeholder: reload first
                raise ContractError(f"request {s.request_id} has KV rows on the host tier; reload them first")
            if self.on_demand:
                if s in verifs:
                    end = s.n_kv + s.round_target + 1
                else:
                    end = (s.n_kv_ub if s.inflight else s.n_kv) + s.phase + 1
                self.pool.ensure_tokens(s.slot, end)
        self.pool.sync_table()
        plan = self._plan_host[j].numpy()
        row = 0
        d_max_keys = 1
        for i, s in enumerate(drafts):
            if s.done or s.phase >= s.round_target:
                raise ContractError(f"request {s.request_id} cannot draft now")
            plan[i] = (s.slot, N.PLAN_DRAFT, row, 1, s.phase, i, )
            # an upper bound while the previous verify's outcome is still in flight
            n_kv = s.n_kv_ub if s.inflight else s.n_kv
            crit = min(compute_budget(n_kv, self.sparsity), n_kv) if s.inflight else s.crit_len
            d_max_keys = max(d_max_keys, crit + s.phase + 1)
            row += 1
        n_draft_rows = row
        v_max_keys, v_max_nq = 1, 1
        vinfo = []
        for m, s in enumerate(verifs):
            if s.done or s.phase != s.round_target:
                raise ContractError(f"request {s.request_id} cannot verify now")
            if s.inflight:
                raise ContractError(f"request {s.request_id}: previous verification not processed yet")
            t = s.round_target + 1
            plan[len(drafts) + m] = (s.slot, N.PLAN_VERIFY, row, t, 0, m)
            v_max_keys = max(v_max_keys, s.n_kv + t)
            v_max_nq = max(v_max_nq, t)
            vinfo.append((s, len(s.drafted), s.kv_len, s.budget))
            row += t
        R = row
        if R == 0:
            return PendingStep(self._iter - 1, j, [], [], 0, 0, None, t_host0, time.perf_counter())
        plan_dev = self._plan_dev[:n_members]
        plan_dev.copy_(self._plan_host[j][:n_members], non_blocking=True)
        K.step_prepare(plan_dev, n_members, self.k, self.crit_cap, self.n_kv_dev, self.last_tok_dev,
                       self.drafted_dev, self.crit_len_dev, self._tok_buf, self._rt_buf, self._rp_buf,
                       self._v_items, self._d_items, self.acc, self.acc.stride(0))
        launches = []
        self.last_events = {}

        def events(kind):
            if not self.attn_events:
                return None
            evs = []
            for _ in range(c.num_layers):
                pair = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for e in pair:
                    e.record()  # materialise the CUDA event; re-recorded around the launch
                evs.append(pair)
            self.last_events[kind] = evs
            return evs

        if verifs:
            launches.append(AttnLaunch(self._v_items, len(verifs), v_max_keys, v_max_nq, acc=self.acc,
                                       acc_row_stride=self.acc_w, acc_shift=self.verify_shift,
                                       timer=self._timer("verify"), events=events("verify")))
        if drafts:  # launch 1: overlaps the verify launch on a low-priority stream
            launches.append(AttnLaunch(self._d_items, len(drafts), d_max_keys, 1, crit=self.crit,
                                       timer=self._timer("draft"), events=events("draft")))
        x = forward_rows(self.model, self.pool, self._tok_buf[:R], self._rt_buf[:R], self._rp_buf[:R], launches)
        targets = self._targets[:R]
        logits = lm_head(self.model, x).contiguous()
        K.argmax_rows(logits, targets)
        if self.keep_logits:   # diagnostics (tools/alpha_margin.py): rows in plan order
            self.last_logits = logits
        sel_rows, sel_kv, sel_slot = self._sel[0], self._sel[1], self._sel[2]
        K.step_commit(plan_dev, n_members, self.k, targets, self.n_kv_dev, self.last_tok_dev, self.drafted_dev,
                      sel_rows, sel_kv, sel_slot, self._res_dev)
        if verifs:
            # K3 straight from the device accept results (engine.py:256-259)
            K.select_critical(self.acc, (self.k + 1) * self.acc.stride(0), self.acc.stride(0), self.verify_shift,
                              sel_rows, sel_kv, self.sparsity, len(verifs), self.imp, self.crit, self.crit_len_dev,
                              req_index=sel_slot)
            self._res_host[j][: len(verifs)].copy_(self._res_dev[: len(verifs)], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev))
        self._ring_ev[j] = ev
        # host mirror of the deterministic part of the state machine
        for s in drafts:
            s.drafted.append(None)   # the token itself lives in drafted_dev until the verify
            s.phase += 1
            s.stats.sparse_forwards += 1
        for s, _, _, _ in vinfo:
            s.n_kv_ub = s.n_kv + s.round_target + 1
            s.inflight = True
            s.drafted, s.phase, s.round_target = [], 0, self.k
        return PendingStep(self._iter - 1, j, vinfo, drafts, R, n_draft_rows, ev, t_host0, time.perf_counter())

    def complete(self, pend: "PendingStep") -> StepResult:
        """Wait for a submitted iteration and apply its verify outcomes on the host:
        emissions (engine.py:126-144), round records, KV length, next critical-set size."""
        if pend.event is None:
            return StepResult({}, 0, 0, 0, 0)
        pend.event.synchronize()
        t_synced = time.perf_counter()
        self.host_times.append((pend.t_launched - pend.t_host0, t_synced - pend.t_host0))
        res = self._res_host[pend.ring][: len(pend.verifs)].numpy()
        emitted = 0
        accepted = {}
        for m, (s, n_drafted, kv_at, budget) in enumerate(pend.verifs):
            a, bonus = int(res[m, 0]), int(res[m, 1])
            drafts_m = [int(t) for t in res[m, 2:2 + n_drafted]]
            s.n_kv += a + 1  # KV rollback: rows beyond n_kv + a are dead
            s.inflight = False
            landed = self._emit(s, drafts_m[:a] + [bonus])
            emitted += landed
            s.stats.emitted_tokens += landed
            s.stats.full_forwards += 1
            s.stats.rounds.append(RoundRecord(len(s.stats.rounds), n_drafted, a, kv_at, budget))
            accepted[s.request_id] = a
            s.budget = compute_budget(s.n_kv, self.sparsity)
            s.crit_len = min(s.budget, s.n_kv)
        self.last_rows = pend.rows
        return StepResult(accepted, emitted, pend.rows, pend.draft_rows, pend.rows - pend.draft_rows)

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
