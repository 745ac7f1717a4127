"""PillarAttn critical-token selection (drop-in for the reference selection.py).

The verification kernel (K2) never materialises logits: it emits, per query
row q and KV position p, acc[q][p] = sum_{layer, head} exp(logit - lse) —
exactly the numerator of the reference's aggregated importance
(selection.py:78-135, 207-218; uniform mean over (layer, query, head) since
every kv group has G heads).  ``AttentionScoreLog`` here holds that
accumulator plus the per-(layer, query, head) lse; ``importance_from_log``
divides by the row count, and ``select_critical_tokens`` is the tie-exact
GPU top-k (K3).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import kernels as K
from .errors import ConfigurationError, ContractError

LSE_TOL = 1e-9


def compute_budget(kv_length: int, sparsity: float) -> int:
    """ceil(s * n - 1e-9) clamped to [1, n]; n = 0 -> 1 (selection.py:167-183).

    Host scalar used to size buffers; the device computes the same IEEE
    expression inside K3 (select.cu budget_of) without FMA contraction."""
    if not (0.0 < sparsity <= 1.0):
        raise ConfigurationError(f"sparsity must be in (0, 1], got {sparsity}")
    if kv_length < 0:
        raise ContractError("kv_length must be non-negative")
    if kv_length == 0:
        return 1
    return max(1, min(math.ceil(sparsity * kv_length - 1e-9), kv_length))


@dataclass(frozen=True)
class CriticalTokenSet:
    """Sorted unique positions a draft may attend to (selection.py:138-164).

    ``positions`` is a host int64 array (API parity); the device copy used by
    the draft kernel is cached in ``device_positions``."""

    positions: np.ndarray
    budget: int
    identified_at: int
    _dev: dict = field(default_factory=dict, compare=False, repr=False)

    def __post_init__(self) -> None:
        pos = self.positions
        if isinstance(pos, torch.Tensor):
            if pos.is_cuda:
                self._dev[pos.device] = pos.to(torch.int32)
            pos = pos.cpu().numpy()
        pos = np.asarray(pos, dtype=np.int64)
        object.__setattr__(self, "positions", pos)
        if pos.ndim != 1:
            raise ContractError("positions must be one-dimensional")
        if pos.size != min(self.budget, self.identified_at):
            raise ContractError("position count must be min(budget, identified_at)")
        if pos.size:
            if pos[0] < 0 or pos[-1] >= self.identified_at:
                raise ContractError("positions must lie in [0, identified_at)")
            if np.any(np.diff(pos) <= 0):
                raise ContractError("positions must be strictly increasing")

    def __len__(self) -> int:
        return int(self.positions.size)

    def device_positions(self, device) -> torch.Tensor:
        device = torch.device(device)
        t = self._dev.get(device)
        if t is None:
            t = torch.as_tensor(self.positions.astype(np.int32), device=device)
            if t.numel() == 0:
                t = torch.zeros(1, dtype=torch.int32, device=device)
            self._dev[device] = t
        return t


def select_critical_tokens(importance, budget: int) -> CriticalTokenSet:
    """Top-``budget`` positions, ties to the lower index, ascending
    (selection.py:186-204).  Runs on the GPU (K3 top-k); float64 inputs are
    selected on their exact bits, float32 inputs on theirs."""
    t = importance if isinstance(importance, torch.Tensor) else torch.as_tensor(np.asarray(importance, dtype=np.float64))
    if t.dim() != 1:
        raise ContractError("importance must be a vector")
    if budget < 1:
        raise ContractError("budget must be at least 1")
    if t.dtype not in (torch.float32, torch.float64):
        t = t.double()
    if not t.is_cuda:
        t = t.cuda()
    if not bool(torch.isfinite(t).all()):
        raise ContractError("importance values must be finite")
    n = t.shape[0]
    take = min(budget, n)
    if n == 0:
        return CriticalTokenSet(positions=np.zeros(0, dtype=np.int64), budget=budget, identified_at=0)
    dev = t.device
    out = torch.empty(1, max(take, 1), dtype=torch.int32, device=dev)
    out_len = torch.empty(1, dtype=torch.int32, device=dev)
    K.topk(t.reshape(1, n).contiguous(), torch.tensor([n], dtype=torch.int32, device=dev),
           torch.tensor([budget], dtype=torch.int32, device=dev), out, out_len)
    return CriticalTokenSet(positions=out[0, :take], budget=budget, identified_at=n)


@dataclass(frozen=True)
class ScoreRow:
    """Logits (Hq, kv_len) + lse (Hq,) of one (layer, query) (selection.py:24-37).
    The hot path never materialises these; device-captured logs build them on demand."""

    logits: object
    lse: object

    def kv_len(self) -> int:
        return int(self.logits.shape[1])


def _as_f64(x) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.float64))
    if not t.is_cuda:
        t = t.cuda()
    return t.double()


class AttentionScoreLog:
    """Score capture of one full-attention forward (selection.py:40-75).

    Two backings share the reference interface (``layers``, ``group_map``,
    ``num_queries``, ``slice_queries``, ``validate``):

    * ``AttentionScoreLog(num_q_heads, num_kv_heads, layers)`` — explicit
      ``layers[l][q]`` ScoreRows, exactly the reference's constructor;
    * ``AttentionScoreLog.from_accumulators(...)`` — what forward_full returns:
      acc (n_queries, n0 + n_queries) int64 fixed point (unit 2^-acc_shift),
      acc[q][p] = sum over layers and q heads of exp(logit - lse) for query q
      (zero where causally hidden), emitted by the verify kernel; lse (layers,
      n_queries, Hq) fp32.  ``layers`` is materialised on first access from the
      per-layer rotated queries and the cache's keys (valid until the cache
      rows [0, n0 + n_queries) are overwritten).
    """

    def __init__(self, num_q_heads: int, num_kv_heads: int, layers: list | None = None):
        self.num_q_heads = num_q_heads
        self.num_kv_heads = num_kv_heads
        self._layers = layers if layers is not None else []
        self.num_layers = len(self._layers)
        self.n0 = 0
        self.acc = None
        self.lse = None
        self.acc_shift = 0
        self._rows_fn = None
        self._nq = len(self._layers[0]) if self._layers else 0
        self._dtype_tol = 0.0

    @classmethod
    def from_accumulators(cls, num_q_heads: int, num_kv_heads: int, num_layers: int, n0: int,
                          acc: torch.Tensor | None, lse: torch.Tensor | None, acc_shift: int = 0,
                          rows_fn=None, n_queries: int | None = None, dtype_tol: float = 0.0):
        log = cls(num_q_heads, num_kv_heads, None)
        log.num_layers = num_layers
        log.n0 = n0
        log.acc, log.lse, log.acc_shift = acc, lse, acc_shift
        log._rows_fn = rows_fn
        full = 0 if acc is None else acc.shape[0]
        log._nq = full if n_queries is None else min(n_queries, full)
        log._dtype_tol = dtype_tol
        return log

    @property
    def captured(self) -> bool:
        return self.acc is not None or bool(self._layers)

    @property
    def layers(self) -> list:
        if self.acc is None:
            if self._layers or self.lse is not None or self.num_layers == 0:
                return self._layers
            return [[] for _ in range(self.num_layers)]   # capture_scores=False
        if self._rows_fn is None:
            raise ContractError("this score log carries accumulators only")
        if not self._layers:
            self._layers = self._rows_fn()
        return [rows[: self._nq] for rows in self._layers]

    def group_map(self) -> np.ndarray:
        return np.arange(self.num_q_heads) // (self.num_q_heads // self.num_kv_heads)

    def num_queries(self) -> int:
        return self._nq

    def slice_queries(self, n: int) -> "AttentionScoreLog":
        """Restrict to the first ``n`` query tokens (selection.py:60-64)."""
        if self.acc is None:
            return AttentionScoreLog(self.num_q_heads, self.num_kv_heads, [rows[:n] for rows in self._layers])
        out = AttentionScoreLog.from_accumulators(self.num_q_heads, self.num_kv_heads, self.num_layers, self.n0,
                                                  self.acc, self.lse, self.acc_shift, self._rows_fn,
                                                  n_queries=min(n, self._nq), dtype_tol=self._dtype_tol)
        out._layers = self._layers
        return out

    def row_kv_len(self, q: int) -> int:
        return self.n0 + q + 1

    def validate(self, tol: float = LSE_TOL) -> None:
        """Every stored lse matches its logit row (selection.py:66-75).  Device-captured
        lse values are computed in the kernel's precision, so the tolerance is at least
        that precision's (1e-4 fp32, 2e-2 bf16 per north_star)."""
        tol = max(tol, self._dtype_tol)
        for rows in self.layers:
            for row in rows:
                lg = _as_f64(row.logits)
                if not bool(torch.isfinite(lg).all()):
                    raise ContractError("score log contains non-finite logits")
                lse = torch.logsumexp(lg, dim=1)
                if float((lse - _as_f64(row.lse)).abs().max()) > tol:
                    raise ContractError("stored lse disagrees with logits")


def rematerialize_scores(log: AttentionScoreLog) -> list:
    """exp(logit - lse) per row, same layers-by-queries nesting (selection.py:78-92)."""
    out = []
    for layer_rows in log.layers:
        cur = []
        for r in layer_rows:
            lg, ls = _as_f64(r.logits), _as_f64(r.lse)
            if not bool(torch.isfinite(lg).all()) or not bool(torch.isfinite(ls).all()):
                raise ContractError("cannot rematerialize non-finite scores")
            cur.append(torch.exp(lg - ls[:, None]))
        out.append(cur)
    return out


def pad_rows(rows: Sequence, length: int) -> list:
    """Right-pad probability rows with zeros to ``length`` (selection.py:95-109)."""
    res = []
    for r in rows:
        if r.shape[-1] > length:
            raise ContractError(f"row covers {r.shape[-1]} positions, beyond target {length}")
        pad = length - r.shape[-1]
        if not pad:
            res.append(r)
        elif isinstance(r, torch.Tensor):
            res.append(torch.nn.functional.pad(r, (0, pad)))
        else:
            res.append(np.pad(r, ((0, 0), (0, pad))))
    return res


def aggregate_scores(scores: Sequence, group_map: Sequence[int]) -> torch.Tensor:
    """Mean over rows, heads within a kv group, then groups (selection.py:112-135); fp64."""
    if len(scores) == 0:
        raise ContractError("aggregate_scores needs at least one row")
    gm = np.asarray(group_map)
    width = scores[0].shape[-1]
    for r in scores:
        if r.ndim != 2 or r.shape[0] != gm.shape[0]:
            raise ContractError("score row shape disagrees with group map")
        if r.shape[-1] != width:
            raise ContractError("inconsistent score row lengths")
    st = torch.stack([_as_f64(r) for r in scores])
    groups = [st[:, torch.as_tensor(gm == g, device=st.device), :].mean(dim=(0, 1)) for g in np.unique(gm).tolist()]
    return torch.stack(groups).mean(dim=0)


def importance_from_log(log: AttentionScoreLog, kv_len: int) -> torch.Tensor:
    """Mean over (layer, surviving query, head) of exp(logit - lse), zero padded to
    ``kv_len`` (selection.py:207-218).  Device fp64 vector.  For device-captured logs
    this is the fixed-point accumulator sum divided by the row count (no logits)."""
    if log.acc is None:
        if not log.captured:
            raise ContractError("score log is empty (capture_scores was off)")
        flat = []
        for layer_rows in rematerialize_scores(log):
            flat.extend(pad_rows(layer_rows, kv_len))
        return aggregate_scores(flat, log.group_map())
    nq = log.num_queries()
    if nq == 0:
        raise ContractError("aggregate_scores needs at least one row")
    if log.row_kv_len(nq - 1) > kv_len:
        raise ContractError(f"row covers {log.row_kv_len(nq - 1)} positions, beyond target {kv_len}")
    out = torch.zeros(kv_len, dtype=torch.float64, device=log.acc.device)
    w = min(kv_len, log.acc.shape[1])
    out[:w] = K.scores_to_float(log.acc[:nq, :w], log.acc_shift).sum(dim=0)
    return out / float(nq * log.num_layers * log.num_q_heads)


def select_from_log(log: AttentionScoreLog, kv_len: int, sparsity: float) -> CriticalTokenSet:
    """Fused refresh (engine.py:147-151): K3 sums the surviving accumulator
    rows, computes the budget on device and selects, in one launch."""
    if log.acc is None:
        return select_critical_tokens(importance_from_log(log, kv_len), compute_budget(kv_len, sparsity))
    nq = log.num_queries()
    if log.row_kv_len(nq - 1) > kv_len:
        raise ContractError("score rows exceed kv_len")
    dev = log.acc.device
    budget = compute_budget(kv_len, sparsity)
    take = min(budget, kv_len)
    acc = log.acc
    if acc.shape[1] < kv_len:
        acc = torch.nn.functional.pad(acc, (0, kv_len - acc.shape[1]))
    imp = torch.empty(1, max(kv_len, 1), dtype=torch.float64, device=dev)
    crit = torch.empty(1, max(take, 1), dtype=torch.int32, device=dev)
    crit_len = torch.empty(1, dtype=torch.int32, device=dev)
    K.select_critical(acc, 0, acc.stride(0), log.acc_shift, torch.tensor([nq], dtype=torch.int32, device=dev),
                      torch.tensor([kv_len], dtype=torch.int32, device=dev), sparsity, 1, imp, crit, crit_len)
    return CriticalTokenSet(positions=crit[0, :take], budget=budget, identified_at=kv_len)
