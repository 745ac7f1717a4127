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
    Only produced by explicit debug capture; the hot path keeps accumulators."""

    logits: torch.Tensor
    lse: torch.Tensor

    def kv_len(self) -> int:
        return int(self.logits.shape[1])


class AttentionScoreLog:
    """Score capture of one full-attention forward.

    acc : (n_queries, n0 + n_queries) fp32, acc[q][p] = sum over layers and
          q heads of exp(logit - lse) for query q (zero where causally hidden)
    lse : (layers, n_queries, Hq) fp32
    """

    def __init__(self, num_q_heads: int, num_kv_heads: int, num_layers: int, n0: int,
                 acc: torch.Tensor | None, lse: torch.Tensor | None, n_queries: int | None = None):
        self.num_q_heads = num_q_heads
        self.num_kv_heads = num_kv_heads
        self.num_layers = num_layers
        self.n0 = n0
        self.acc = acc
        self.lse = lse
        full = 0 if acc is None else acc.shape[0]
        self._nq = full if n_queries is None else n_queries

    def group_map(self) -> np.ndarray:
        return np.arange(self.num_q_heads) // (self.num_q_heads // self.num_kv_heads)

    def num_queries(self) -> int:
        return self._nq

    @property
    def captured(self) -> bool:
        return self.acc is not None

    def slice_queries(self, n: int) -> "AttentionScoreLog":
        """Restrict to the first ``n`` query tokens (selection.py:60-64)."""
        return AttentionScoreLog(self.num_q_heads, self.num_kv_heads, self.num_layers, self.n0, self.acc,
                                 self.lse, n_queries=min(n, self._nq))

    def row_kv_len(self, q: int) -> int:
        return self.n0 + q + 1


def importance_from_log(log: AttentionScoreLog, kv_len: int) -> torch.Tensor:
    """Mean over (layer, surviving query, head) of exp(logit - lse), zero
    padded to ``kv_len`` (selection.py:207-218).  Device fp32 vector."""
    if not log.captured:
        raise ContractError("score log is empty (capture_scores was off)")
    nq = log.num_queries()
    if nq == 0:
        raise ContractError("aggregate_scores needs at least one row")
    if log.row_kv_len(nq - 1) > kv_len:
        raise ContractError(f"row covers {log.row_kv_len(nq - 1)} positions, beyond target {kv_len}")
    out = torch.zeros(kv_len, dtype=torch.float32, device=log.acc.device)
    w = min(kv_len, log.acc.shape[1])
    out[:w] = log.acc[:nq, :w].sum(dim=0)
    return out / float(nq * log.num_layers * log.num_q_heads)


def select_from_log(log: AttentionScoreLog, kv_len: int, sparsity: float) -> CriticalTokenSet:
    """Fused refresh (engine.py:147-151): K3 sums the surviving accumulator
    rows, computes the budget on device and selects, in one launch."""
    nq = log.num_queries()
    if log.row_kv_len(nq - 1) > kv_len:
        raise ContractError("score rows exceed kv_len")
    dev = log.acc.device
    budget = compute_budget(kv_len, sparsity)
    take = min(budget, kv_len)
    acc = log.acc
    if acc.shape[1] < kv_len:
        acc = torch.nn.functional.pad(acc, (0, kv_len - acc.shape[1]))
    imp = torch.empty(1, max(kv_len, 1), dtype=torch.float32, device=dev)
    crit = torch.empty(1, max(take, 1), dtype=torch.int32, device=dev)
    crit_len = torch.empty(1, dtype=torch.int32, device=dev)
    K.select_critical(acc, 0, acc.stride(0), torch.tensor([nq], dtype=torch.int32, device=dev),
                      torch.tensor([kv_len], dtype=torch.int32, device=dev), sparsity, 1, imp, crit, crit_len)
    return CriticalTokenSet(positions=crit[0, :take], budget=budget, identified_at=kv_len)


# -- array utilities kept for API parity (device torch ops on caller data) ----------


def rematerialize_scores(rows: Sequence[Sequence[ScoreRow]]) -> list:
    """exp(logit - lse) per row (selection.py:78-92)."""
    out = []
    for layer_rows in rows:
        cur = []
        for r in layer_rows:
            if not bool(torch.isfinite(r.logits).all()) or not bool(torch.isfinite(r.lse).all()):
                raise ContractError("cannot rematerialize non-finite scores")
            cur.append(torch.exp(r.logits - r.lse[:, None]))
        out.append(cur)
    return out


def pad_rows(rows: Sequence[torch.Tensor], length: int) -> list:
    """Right-pad with zeros to ``length`` (selection.py:95-109)."""
    res = []
    for r in rows:
        if r.shape[-1] > length:
            raise ContractError(f"row covers {r.shape[-1]} positions, beyond target {length}")
        res.append(torch.nn.functional.pad(r, (0, length - r.shape[-1])))
    return res


def aggregate_scores(scores: Sequence[torch.Tensor], group_map: Sequence[int]) -> torch.Tensor:
    """Mean over rows, heads within a kv group, then groups (selection.py:112-135)."""
    if len(scores) == 0:
        raise ContractError("aggregate_scores needs at least one row")
    gm = torch.as_tensor(np.asarray(group_map))
    width = scores[0].shape[-1]
    for r in scores:
        if r.dim() != 2 or r.shape[0] != gm.shape[0]:
            raise ContractError("score row shape disagrees with group map")
        if r.shape[-1] != width:
            raise ContractError("inconsistent score row lengths")
    st = torch.stack(list(scores))
    groups = [st[:, (gm == g).to(st.device), :].mean(dim=(0, 1)) for g in torch.unique(gm).tolist()]
    return torch.stack(groups).mean(dim=0)
