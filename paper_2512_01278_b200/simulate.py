"""Token-level unified serving loop on the GPU (drop-in for the reference's
``run_token_sim``, simulate.py:271-548).

Per iteration, exactly the reference's control flow: transfer step, admission
in arrival order with PhaseBuckets placement and a shortened first round,
prompt grants + prefill, candidate list, ``form_batch`` (delayed-verification
stalls), one KvPool page per draft and per verify, ``free_tail`` of rejected
drafts, ``step_pipeline`` and ``KvPool.check``.  The difference is the
execution: all prefills of an iteration run as one batched prompt pass and
all draft / verify members as ONE batched forward (serving.BatchedDecoder),
and latency is the measured GPU time of that forward instead of an analytic
cost model (the cost-level simulator is out of scope).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import torch

from .engine import DecodeRequest
from .errors import ConfigurationError, SimulationError
from .kvpool import KvPolicy, KvPool, utilization_report
from .model import ModelConfig, ToyModel, init_model
from .scheduler import (BatchCandidate, PhaseBuckets, PipelineMode, PipelineSlot, SchedPolicy, assign_new_request,
                        first_round_draft_len, form_batch, step_pipeline)
from .selection import compute_budget
from .serving import BatchedDecoder
from .workload import WorkloadSpec, generate_workload, synthetic_prompt


@dataclass(frozen=True)
class KvPoolConfig:
    capacity_pages: int
    page_bytes: int
    chunk_pages: int = 64
    pcie_gbps: float = 16.0
    policy: KvPolicy = KvPolicy.OFFLOAD

    def __post_init__(self) -> None:
        if self.capacity_pages < 1:
            raise ConfigurationError("capacity_pages must be at least 1")
        if self.page_bytes < 1:
            raise ConfigurationError("page_bytes must be at least 1")
        if self.chunk_pages < 1:
            raise ConfigurationError("chunk_pages must be at least 1")
        if self.pcie_gbps <= 0:
            raise ConfigurationError("pcie_gbps must be positive")


@dataclass(frozen=True)
class SimConfig:
    k: int
    alpha: float
    sparsity: float
    max_batch: int
    sched_policy: SchedPolicy = SchedPolicy.UNIFIED
    pipeline: PipelineMode = PipelineMode.DELAYED
    cpu_ms_per_verify: float = 0.0
    max_iterations: int = 1_000_000

    def __post_init__(self) -> None:
        if self.k < 1:
            raise ConfigurationError("k must be at least 1")
        if not 0.0 <= self.alpha <= 1.0:
            raise ConfigurationError("alpha must lie in [0, 1]")
        if not 0.0 < self.sparsity <= 1.0:
            raise ConfigurationError("sparsity must lie in (0, 1]")
        if self.max_batch < 1:
            raise ConfigurationError("max_batch must be at least 1")
        if self.cpu_ms_per_verify < 0:
            raise ConfigurationError("cpu_ms_per_verify cannot be negative")


@dataclass(frozen=True)
class IterationRow:
    iteration: int
    gemm_tokens: int
    attn_bytes: int
    latency_ms: float
    device_util: float
    offloaded_pages: int
    stalled_requests: int


ITERATION_CSV_COLUMNS = ("iteration", "gemm_tokens", "attn_bytes", "latency_ms", "device_util",
                         "offloaded_pages", "stalled_requests")


@dataclass(frozen=True)
class Breakdown:
    cpu_ms: float
    attn_ms: float
    gemm_ms: float
    other_ms: float

    @property
    def total_ms(self) -> float:
        return self.cpu_ms + self.attn_ms + self.gemm_ms + self.other_ms


@dataclass(frozen=True)
class RequestSummary:
    request_id: int
    emitted: int
    rounds: int
    stall_absences: int
    pressure_absences: int
    accepted_total: int
    drafted_total: int


@dataclass(frozen=True)
class SimReport:
    level: str
    total_ms: float
    emitted_tokens: int
    tokens_per_second: float
    iterations: tuple
    breakdown: Breakdown
    eta: float
    recomputation_ratio: float
    requests: tuple
    realized_alpha: float | None = None
    acceptance_histogram: dict | None = None
    outputs: dict | None = None


@dataclass
class _Live:
    req: object
    round_target: int
    prompt_granted: bool = False
    drafts_done: int = 0
    rounds: int = 0
    emitted: int = 0
    stall_absences: int = 0
    pressure_absences: int = 0
    accepted_total: int = 0
    drafted_total: int = 0
    done: bool = False


def run_token_sim(workload: WorkloadSpec, model_config: ModelConfig, cfg: SimConfig, kv_cfg: KvPoolConfig,
                  params=None, *, model: ToyModel | None = None, dtype: torch.dtype = torch.float32,
                  check_lossless: bool = True) -> SimReport:
    """Serve ``workload`` with the real model on the GPU; returns the same
    report fields as the reference.  ``params`` (cost model) is accepted for
    signature parity and ignored: latency is measured.  Like the reference
    (simulate.py:245-248), every completed request is checked against the
    autoregressive oracle (greedy_decode on the same model) unless
    ``check_lossless=False``."""
    if model is None:
        model = init_model(model_config, dtype=dtype)
    if kv_cfg.policy is KvPolicy.PREEMPT:
        raise ConfigurationError("preemption resume is cost-level only")
    requests = generate_workload(workload)
    k = cfg.k
    max_len = max((r.input_len + r.output_len for r in requests), default=1)
    # physical pages follow KvPool's logical accounting: granted as positions are written,
    # sized to the pool's capacity (+ one partly filled page and the k+1 in-flight
    # positions per request slot)
    dec = BatchedDecoder(model, k, cfg.sparsity, max_requests=cfg.max_batch, max_seq_len=max_len,
                         paging="on_demand",
                         pool_tokens=kv_cfg.capacity_pages + cfg.max_batch * (16 + k + 1))
    pool = KvPool(kv_cfg.capacity_pages, kv_cfg.page_bytes, chunk_pages=kv_cfg.chunk_pages, policy=kv_cfg.policy)
    waiting = sorted(requests, key=lambda r: (r.arrival_ms, r.request_id))
    lives: dict = {}
    finished: dict = {}
    outputs: dict = {}
    pipeline = PipelineSlot()
    histogram: dict = {}
    rows, snapshots = [], []
    sim_time = 0.0
    pressure_last = False
    gpu_total = 0.0
    host_pages: dict = {}  # request -> token pages on the host tier after the last transfer step

    def complete(rid):
        host_pages.pop(rid, None)
        pool.release(rid)
        seq = dec.seqs[rid]
        outputs[rid] = list(seq.committed)
        if check_lossless:
            from .engine import greedy_decode
            want = greedy_decode(model, seq.prompt, seq.max_output, seq.eos_token)
            if want != seq.committed:
                raise SimulationError(f"request {rid}: speculative output diverged from the autoregressive oracle")
        dec.release(rid)
        finished[rid] = lives.pop(rid)

    def phase_of(lv):
        return k - (lv.round_target - lv.drafts_done)

    for iteration in range(cfg.max_iterations):
        if not lives and not waiting:
            break
        if not lives and waiting[0].arrival_ms > sim_time:
            sim_time = waiting[0].arrival_ms
        pool.step(kv_cfg.capacity_pages, kv_cfg.capacity_pages, allow_reload=not pressure_last)
        # host tier (kvpool.py:213-237,272-311): the pages the pool moved this iteration
        # really move; K/V rows of offloaded token pages go to pinned host memory (their
        # device pages are returned) and come back on reload
        for rid in list(dec.seqs):
            now = set(pool.host_pages_of(rid))
            before = host_pages.get(rid, set())
            if now - before:
                dec.offload_positions(rid, now - before)
            if before - now:
                dec.reload_positions(rid, before - now)
            host_pages[rid] = now
        pressure_now = False
        while waiting and waiting[0].arrival_ms <= sim_time and len(lives) < cfg.max_batch:
            req = waiting[0]
            if not pool.admit(req.request_id, expected_total=req.input_len + req.output_len + k + 1):
                break
            waiting.pop(0)
            counts = [0] * (k + 1)
            for lv in lives.values():
                counts[phase_of(lv)] += 1
            phase = assign_new_request(PhaseBuckets(k=k, counts=counts), cfg.sched_policy)
            lives[req.request_id] = _Live(req=req, round_target=first_round_draft_len(k, phase))
        to_prefill = []
        for rid, lv in list(lives.items()):
            if lv.prompt_granted:
                continue
            res = pool.allocate(rid, lv.req.input_len + lv.emitted, iteration=iteration)
            if not res.granted:
                pressure_now = True
                continue
            lv.prompt_granted = True
            if lv.emitted == 0:
                to_prefill.append(lv)
        t0 = time.perf_counter()
        if to_prefill:
            reqs = [DecodeRequest(lv.req.request_id, synthetic_prompt(workload.seed, lv.req.request_id,
                                                                      lv.req.input_len, model.config.vocab_size),
                                  lv.req.output_len) for lv in to_prefill]
            for lv, seq in zip(to_prefill, dec.prefill(reqs)):
                seq.round_target = lv.round_target
                lv.emitted = len(seq.committed)
                lv.done = seq.done
                if lv.done:
                    complete(lv.req.request_id)
        cands, by_id = [], {}
        for rid, lv in lives.items():
            if not lv.prompt_granted or not pool.is_schedulable(rid):
                continue
            kv = lv.req.input_len + lv.emitted
            c = BatchCandidate(rid, due_verify=lv.drafts_done == lv.round_target, verify_tokens=lv.round_target + 1,
                               attn_pages_draft=compute_budget(kv, cfg.sparsity) + lv.drafts_done + 1,
                               attn_pages_verify=kv + lv.round_target + 1)
            cands.append(c)
            by_id[rid] = c
        planned, stalled_now = form_batch(cands, pipeline.stalled_verifications, cfg.pipeline)
        for rid in stalled_now:
            lives[rid].stall_absences += 1
        ex_d, ex_v = [], []
        attn_pages = 0
        for rid in planned.draft_members:
            if pool.allocate(rid, 1, iteration=iteration).granted:
                ex_d.append(rid)
                attn_pages += by_id[rid].attn_pages_draft
            else:
                pressure_now = True
                lives[rid].pressure_absences += 1
        for rid in planned.verify_members:
            if pool.allocate(rid, 1, iteration=iteration).granted:
                ex_v.append(rid)
                attn_pages += by_id[rid].attn_pages_verify
            else:
                pressure_now = True
                lives[rid].pressure_absences += 1
        if not ex_d and not ex_v and not to_prefill and not stalled_now and not pressure_now \
                and not pool.transfers_pending and lives and not waiting:
            # deadlock guard (simulate.py:462-463): nothing runnable and nothing in flight
            raise SimulationError("no schedulable work and no pending transfers")
        result = dec.step(ex_d, ex_v)
        torch.cuda.synchronize()
        latency = (time.perf_counter() - t0) * 1000.0
        gpu_total += latency
        for rid in ex_d:
            lives[rid].drafts_done += 1
            lives[rid].drafted_total += 1
        verify_tokens = 0
        for rid in ex_v:
            lv = lives[rid]
            a = result.accepted[rid]
            target = lv.round_target
            pool.free_tail(rid, target - a)
            seq = dec.seqs[rid]
            dec.pool.shrink_row(seq.slot, seq.n_kv + 1)  # rejected drafts' whole pages
            lv.emitted = len(seq.committed)
            lv.done = seq.done
            lv.accepted_total += a
            lv.rounds += 1
            lv.drafts_done = 0
            lv.round_target = k
            histogram[a] = histogram.get(a, 0) + 1
            verify_tokens += target + 1
            if lv.done:
                complete(rid)
        pipeline = step_pipeline(pipeline, ex_v if cfg.pipeline is PipelineMode.DELAYED else [],
                                 pipeline.stalled_verifications)
        sim_time += latency
        pressure_last = pressure_now
        rows.append(IterationRow(iteration, len(ex_d) + verify_tokens, attn_pages * kv_cfg.page_bytes, latency,
                                 pool.utilization, pool.offloaded_pages, len(stalled_now)))
        snapshots.append(pool.snapshot(iteration))
        pool.check()
    else:
        raise SimulationError(f"no completion within {cfg.max_iterations} iterations")

    run_token_sim.last_transfer_bytes = (dec.offloaded_bytes, dec.reloaded_bytes)
    emitted = sum(lv.emitted for lv in finished.values())
    drafted = sum(lv.drafted_total for lv in finished.values())
    accepted = sum(lv.accepted_total for lv in finished.values())
    return SimReport(
        level="token", total_ms=sim_time, emitted_tokens=emitted,
        tokens_per_second=emitted / (sim_time / 1000.0) if sim_time > 0 else 0.0, iterations=tuple(rows),
        breakdown=Breakdown(cpu_ms=0.0, attn_ms=0.0, gemm_ms=0.0, other_ms=gpu_total), eta=0.0,
        recomputation_ratio=utilization_report(snapshots).recomputation_ratio,
        requests=tuple(RequestSummary(rid, lv.emitted, lv.rounds, lv.stall_absences, lv.pressure_absences,
                                      lv.accepted_total, lv.drafted_total) for rid, lv in sorted(finished.items())),
        realized_alpha=(accepted / drafted if drafted else None), acceptance_histogram=dict(sorted(histogram.items())),
        outputs=outputs)
