"""Toy decoder (the reference's oracle architecture) on the B200, and the
drop-in attention operators.

Same public names as the reference model.py: ``ModelConfig``, ``ToyModel``,
``init_model``, ``plant_attention_concentration``, ``KVEntry``, ``KvCache``,
``forward_full``, ``forward_sparse``, ``greedy_token``.

Architecture (model.py:1-17): pre-norm GQA blocks, RMSNorm without gain
(model.py:225), NeoX RoPE base 1e4 (model.py:212-222), tanh MLP of width 2h
(model.py:181,336), tied embedding / LM head (model.py:339), 1/sqrt(d) logit
scale (model.py:245), q head h -> kv head h // G (model.py:244).

Linear layers run on torch.matmul (cuBLAS; TF32 disabled in fp32 parity
mode).  RoPE + KV append (K5) and attention (K1/K2) are the in-tree sm_100a
kernels; there is no CPU path.
"""

from __future__ import annotations

import ctypes

import math
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from . import kernels as K
from .errors import ConfigurationError, ContractError
from .paged import PagedKvPool
from .selection import AttentionScoreLog, CriticalTokenSet, ScoreRow

INIT_SCALE = 0.08   # model.py:31
RMS_EPS = 1e-6      # model.py:32
ROPE_BASE = 10000.0  # model.py:33


@dataclass(frozen=True)
class ModelConfig:
    """Shape and seed (model.py:36-74). hidden_dim is pinned to Hq * d."""

    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    vocab_size: int
    seed: int = 0
    hidden_dim: int | None = None

    def __post_init__(self) -> None:
        if min(self.num_layers, self.num_q_heads, self.num_kv_heads, self.head_dim) < 1:
            raise ConfigurationError("model dimensions must be at least 1")
        if self.vocab_size < 2:
            raise ConfigurationError("vocab_size must be at least 2")
        if self.num_q_heads % self.num_kv_heads:
            raise ConfigurationError(f"num_kv_heads={self.num_kv_heads} must divide num_q_heads={self.num_q_heads}")
        if self.head_dim % 2:
            raise ConfigurationError("head_dim must be even for rotary mixing")
        want = self.num_q_heads * self.head_dim
        if self.hidden_dim is None:
            object.__setattr__(self, "hidden_dim", want)
        elif self.hidden_dim != want:
            raise ConfigurationError(f"hidden_dim must equal num_q_heads * head_dim = {want}")

    @property
    def group_size(self) -> int:
        return self.num_q_heads // self.num_kv_heads


@dataclass(frozen=True)
class PlantedConcentration:
    """+bonus on listed positions for every layer/head/query (model.py:87-97)."""

    positions: tuple
    bonus: float = 2000.0


@dataclass(frozen=True)
class LayerWeights:
    """Views of one layer's matrices, (in, out) layout as the reference."""

    mlp_in: torch.Tensor
    mlp_out: torch.Tensor
    wk: torch.Tensor
    wo: torch.Tensor
    wq: torch.Tensor
    wv: torch.Tensor


class ToyModel:
    """Device-resident weights.  ``w_qkv[l]`` = [wq | wk | wv] (h, (Hq+2Hkv)d); every
    layer matrix is stored [out][in] and exposed as an [in][out] transposed view
    so one GEMM feeds the RoPE/KV-append kernel."""

    def __init__(self, config: ModelConfig, embedding: torch.Tensor, w_qkv, wo, mlp_in, mlp_out,
                 planted: PlantedConcentration | None = None):
        self.config = config
        self.embedding = embedding
        self.w_qkv = list(w_qkv)
        self.wo = list(wo)
        self.mlp_in = list(mlp_in)
        self.mlp_out = list(mlp_out)
        self.planted = planted
        self.dtype = embedding.dtype
        self.device = embedding.device
        self.planted_dev = None
        if planted is not None and planted.positions:
            self.planted_dev = torch.tensor(planted.positions, dtype=torch.int32, device=self.device)

    @property
    def layers(self) -> tuple:
        c = self.config
        qd, kd = c.num_q_heads * c.head_dim, c.num_kv_heads * c.head_dim
        return tuple(
            LayerWeights(mlp_in=self.mlp_in[l], mlp_out=self.mlp_out[l], wk=w[:, qd:qd + kd], wo=self.wo[l],
                         wq=w[:, :qd], wv=w[:, qd + kd:])
            for l, w in enumerate(self.w_qkv)
        )

    @property
    def planted_bonus(self) -> float:
        return 0.0 if self.planted is None else float(self.planted.bonus)

    def with_planted(self, planted: PlantedConcentration | None) -> "ToyModel":
        return ToyModel(self.config, self.embedding, self.w_qkv, self.wo, self.mlp_in, self.mlp_out, planted)


def init_model(config: ModelConfig, dtype: torch.dtype = torch.float32, device="cuda",
               fast_init: bool = False) -> ToyModel:
    """Weights ~ N(0, 0.08) drawn exactly like the reference (model.py:171-195):
    SFC64(seed), embedding first, then per layer mlp_in, mlp_out, wk, wo, wq,
    wv, each row-major.  Every matrix is converted and uploaded as soon as it
    is drawn so host memory stays bounded.

    ``fast_init=True`` draws the same shapes from a seeded on-device torch
    generator instead (benchmark-scale models: identical architecture, not
    bit-identical values)."""
    dev = torch.device(device)
    h = config.hidden_dim
    kvw = config.num_kv_heads * config.head_dim
    shapes = [("mlp_in", (h, 2 * h)), ("mlp_out", (2 * h, h)), ("wk", (h, kvw)), ("wo", (h, h)),
              ("wq", (h, h)), ("wv", (h, kvw))]
    if fast_init:
        gen = torch.Generator(device=dev)
        gen.manual_seed(config.seed)

        def draw(shape):
            return (torch.randn(shape, generator=gen, device=dev, dtype=torch.float32) * INIT_SCALE).to(dtype)
    else:
        rng = np.random.Generator(np.random.SFC64(config.seed))

        def draw(shape):
            return torch.from_numpy(rng.normal(0.0, INIT_SCALE, shape)).to(device=dev, dtype=dtype)

    emb = draw((config.vocab_size, h))
    w_qkv, wo, mlp_in, mlp_out = [], [], [], []
    def out_major(w: torch.Tensor) -> torch.Tensor:
        # stored [out][in] (nn.Linear layout: the GEMMs run cuBLAS's TN form), exposed as the
        # reference's [in][out] matrix through a transposed view (same values)
        return w.t().contiguous().t()

    for _ in range(config.num_layers):
        m = {name: draw(shape) for name, shape in shapes}
        w_qkv.append(out_major(torch.cat([m["wq"], m["wk"], m["wv"]], dim=1)))
        wo.append(out_major(m["wo"]))
        mlp_in.append(out_major(m["mlp_in"]))
        mlp_out.append(out_major(m["mlp_out"]))
        del m
    return ToyModel(config, emb, w_qkv, wo, mlp_in, mlp_out)


def plant_attention_concentration(model: ToyModel, positions: Sequence[int], bonus: float = 2000.0) -> ToyModel:
    """model.py:198-209 (weights are shared, not copied)."""
    pos = tuple(sorted(int(p) for p in positions))
    if len(pos) != len(set(pos)) or (pos and pos[0] < 0):
        raise ContractError("planted positions must be unique and non-negative")
    return model.with_planted(PlantedConcentration(positions=pos, bonus=bonus))


# ---------------------------------------------------------------------------------
# batched forward core (shared by the drop-in operators and the batched decoder)
# ---------------------------------------------------------------------------------


def rmsnorm(x: torch.Tensor) -> torch.Tensor:
    """model.py:225-226 (fp32 statistics); torch reference form for tests."""
    return x * torch.rsqrt(torch.mean(x * x, dim=-1, keepdim=True) + RMS_EPS)


def _mm(a: torch.Tensor, b: torch.Tensor, out_f32: bool) -> torch.Tensor:
    if a.dtype == torch.float32 or not out_f32:
        return torch.mm(a, b)
    return torch.mm(a, b, out_dtype=torch.float32)


_ADDMM_MIXED = None


def _residual_add(x: torch.Tensor, a: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """x + a @ w accumulated into the fp32 residual stream in one cuBLAS call
    (beta = 1) when the torch build supports the mixed-dtype epilogue."""
    global _ADDMM_MIXED
    if a.dtype == torch.float32:
        return x.addmm_(a, w)
    if _ADDMM_MIXED is not False:
        try:
            y = torch.addmm(x, a, w, out_dtype=torch.float32)
            _ADDMM_MIXED = True
            return y
        except (RuntimeError, TypeError):
            _ADDMM_MIXED = False
    return x.add_(torch.mm(a, w, out_dtype=torch.float32))


@dataclass
class AttnLaunch:
    """One sd_attention launch over a homogeneous group of work items."""

    items: torch.Tensor           # device int32 [n, ITEM_FIELDS]
    num_items: int
    max_keys: int
    max_nq: int
    crit: torch.Tensor | None = None
    acc: torch.Tensor | None = None  # int64 fixed-point score accumulators (unit 2^-acc_shift)
    acc_row_stride: int = 0
    acc_shift: int = 0
    timer: object | None = None   # optional callable(start: bool) for per-launch timing (torch loop)
    events: list | None = None    # optional [(start, end) torch.cuda.Event] per layer (native loop)


# Overlapping the verify and draft launches of a layer on two streams was measured SLOWER
# (1810 vs 1947 tokens/s on configs[1]: the two kernels starve each other's CTAs), so off.
CONCURRENT_LAUNCHES = False
_SIDE: dict = {}


def _side_stream(device) -> torch.cuda.Stream:
    key = torch.device(device)
    st = _SIDE.get(key)
    if st is None:
        st = torch.cuda.Stream(device=key)
        _SIDE[key] = st
    return st


def forward_rows(model: ToyModel, pool: PagedKvPool, tokens: torch.Tensor, row_table: torch.Tensor,
                 row_pos: torch.Tensor, launches: Sequence[AttnLaunch], lse_out: torch.Tensor | None = None,
                 force_generic: bool = False, q_trace: list | None = None) -> torch.Tensor:
    """Run every layer for R rows at once and return the final hidden (R, h) fp32.

    Row r is token ``tokens[r]`` at absolute position ``row_pos[r]`` of the
    request mapped to block-table row ``row_table[r]``; its K/V are written
    into the pool before attention (K5), so a verify window attends causally to
    its own earlier rows exactly like the reference's token-at-a-time loop
    (model.py:318-340), and a draft row attends to critical U fresh U self
    (model.py:360-380).  Per layer: norm (glue) -> QKV GEMM -> K5 -> K1/K2 ->
    out-proj GEMM (+residual) -> norm -> MLP-in GEMM -> tanh -> MLP-out GEMM
    (+residual)."""
    c = model.config
    R = tokens.shape[0]
    Hq, d = c.num_q_heads, c.head_dim
    dt = model.dtype
    x = model.embedding.index_select(0, tokens.long()).float()
    if (NATIVE_FORWARD and dt == torch.bfloat16 and lse_out is None and not force_generic and q_trace is None
            and all(ln.timer is None for ln in launches)):
        return _forward_native(model, pool, tokens, row_table, row_pos, launches, x)
    if any(ln.events is not None for ln in launches):
        raise ContractError("per-launch events are recorded by the native (bf16) layer loop only")
    hn = torch.empty(R, c.hidden_dim, dtype=dt, device=model.device)
    q_buf = torch.empty(R, Hq, d, dtype=dt, device=model.device)
    ctx = torch.empty(R, Hq, d, dtype=dt, device=model.device)
    main = torch.cuda.current_stream(model.device)
    side = (_side_stream(model.device) if len(launches) > 1 and CONCURRENT_LAUNCHES and not force_generic
            and model.dtype == torch.bfloat16 else None)
    ev_in = torch.cuda.Event() if side is not None else None
    ev_out = torch.cuda.Event() if side is not None else None

    def attend(ln, l):
        if ln.timer is not None:
            ln.timer(True)
        K.attention(q_buf, ctx, pool, l, ln.items, ln.num_items, ln.max_keys, ln.max_nq, Hq,
                    crit=ln.crit, lse=None if lse_out is None else lse_out[l], acc=ln.acc,
                    acc_row_stride=ln.acc_row_stride, acc_shift=ln.acc_shift, planted=model.planted_dev,
                    planted_bonus=model.planted_bonus, force_generic=force_generic)
        if ln.timer is not None:
            ln.timer(False)

    for l in range(c.num_layers):
        K.rmsnorm_cast(x, hn, RMS_EPS)
        qkv = torch.mm(hn, model.w_qkv[l])
        K.rope_kv_write(qkv, row_table, row_pos, pool, l, Hq, q_buf)
        if q_trace is not None:
            q_trace.append(q_buf.clone())
        if side is None:
            for ln in launches:
                attend(ln, l)
        else:
            # the launches touch disjoint rows of q / ctx (and disjoint score rows): the later
            # ones (draft items) run on a side stream and fill the tail waves of the first
            ev_in.record(main)
            side.wait_event(ev_in)
            with torch.cuda.stream(side):
                for ln in launches[1:]:
                    attend(ln, l)
            ev_out.record(side)
            attend(launches[0], l)
            main.wait_event(ev_out)
        x = _residual_add(x, ctx.view(R, Hq * d), model.wo[l])
        K.rmsnorm_cast(x, hn, RMS_EPS)
        hm = torch.mm(hn, model.mlp_in[l])
        torch.tanh_(hm)
        x = _residual_add(x, hm, model.mlp_out[l])
    return x


NATIVE_FORWARD = True  # bf16: the layer loop runs in the library (sd_forward_layers), one host call
# verify (K2) and draft (K1) launches of a layer concurrently on priority streams (K1's CTAs
# fill K2's tail waves): configs[1] 2970 vs 2907 tok/s serial with the TMA K2 producer and
# the four-warp K1 producer (round 2; round 1's kernels measured 2823 vs 2858), so on unless
# SD_ATTN_OVERLAP=0
OVERLAP_ATTENTION = os.environ.get("SD_ATTN_OVERLAP", "1") == "1"
# f3: verify and draft work of a layer in ONE launch (csrc/attn_umma.cu launch_attn_pair)
FUSED_ATTENTION = os.environ.get("SD_ATTN_FUSED", "0") == "1"
# the native layer loop captured and launched as one CUDA graph (csrc/forward.cu
# launch_as_graph: cached executable updated in place per call) unless SD_FORWARD_GRAPH=0
FORWARD_GRAPH = os.environ.get("SD_FORWARD_GRAPH", "1") == "1"
# query rows (tokens x GQA group) per attention work item for multi-token windows (prefill,
# forward_full): <= 48 keeps the tcgen05 verify kernel at two CTAs per SM
ITEM_ROWS = 48


def _forward_native(model: ToyModel, pool: PagedKvPool, tokens, row_table, row_pos, launches, x):
    """forward_rows for bf16 pools through sd_forward_layers: the same per-layer launches
    (glue, cuBLAS GEMMs, K5, K1/K2) issued from C++ instead of Python."""
    c = model.config
    R = tokens.shape[0]
    Hq, d, h = c.num_q_heads, c.head_dim, c.hidden_dim
    dev, dt = model.device, model.dtype
    lib = N.lib()
    wts = getattr(model, "_native_weights", None)
    if wts is None:
        wts = (N.LayerWeights * c.num_layers)()
        for l in range(c.num_layers):
            wts[l].w_qkv = model.w_qkv[l].data_ptr()
            wts[l].wo = model.wo[l].data_ptr()
            wts[l].mlp_in = model.mlp_in[l].data_ptr()
            wts[l].mlp_out = model.mlp_out[l].data_ptr()
        model._native_weights = wts
    desc = pool.desc()
    descs = (N.AttnLaunchDesc * max(1, len(launches)))()
    need = 0
    for i, ln in enumerate(launches):
        descs[i].items = ln.items.data_ptr()
        descs[i].num_items = ln.num_items
        descs[i].max_keys = ln.max_keys
        descs[i].max_nq = ln.max_nq
        descs[i].crit = N.ptr(ln.crit)
        descs[i].acc = N.ptr(ln.acc)
        descs[i].acc_row_stride = ln.acc_row_stride
        descs[i].acc_shift = ln.acc_shift
        need = max(need, lib.sd_attention_workspace_bytes(ln.num_items, ln.max_keys, ln.max_nq, Hq,
                                                          ctypes.byref(desc)))
    need = lib.sd_forward_workspace_bytes(R, d, need)   # + the per-forward RoPE table
    ws = K._zeroed_workspace(need, dev) if need > 0 else None
    qkv_w = (Hq + 2 * c.num_kv_heads) * d
    hn = torch.empty(R, h, dtype=dt, device=dev)
    qkv = torch.empty(R, qkv_w, dtype=dt, device=dev)
    q = torch.empty(R, Hq, d, dtype=dt, device=dev)
    ctx = torch.empty(R, Hq, d, dtype=dt, device=dev)
    hm = torch.empty(R, 2 * h, dtype=dt, device=dev)
    n_planted = 0 if model.planted_dev is None else model.planted_dev.numel()
    ev_arr = None
    if any(ln.events is not None for ln in launches):
        # cudaEvent_t pairs [layer][launch][2] recorded around each attention launch
        ev_arr = (ctypes.c_void_p * (2 * c.num_layers * len(launches)))()
        for i, ln in enumerate(launches):
            if ln.events is None:
                continue
            for l, (e0, e1) in enumerate(ln.events):
                ev_arr[2 * (l * len(launches) + i)] = e0.cuda_event
                ev_arr[2 * (l * len(launches) + i) + 1] = e1.cuda_event
    flags = (0 if OVERLAP_ATTENTION else 1) | (2 if FUSED_ATTENTION else 0) | (8 if FORWARD_GRAPH else 0)
    N.check(lib.sd_forward_layers(wts, c.num_layers, x.data_ptr(), hn.data_ptr(), qkv.data_ptr(), q.data_ptr(),
                                  ctx.data_ptr(), hm.data_ptr(), R, h, Hq, row_table.data_ptr(), row_pos.data_ptr(),
                                  ctypes.byref(desc), descs, len(launches), N.ptr(model.planted_dev), n_planted,
                                  model.planted_bonus, 1.0 / math.sqrt(d), RMS_EPS, N.ptr(ws),
                                  0 if ws is None else ws.numel(), ev_arr, flags, N.stream_handle()),
            "sd_forward_layers")
    return x


def lm_head(model: ToyModel, x: torch.Tensor) -> torch.Tensor:
    """logits = E . rmsnorm(x) (model.py:339), fp32 output."""
    hn = K.rmsnorm_cast(x.contiguous(), torch.empty(x.shape, dtype=model.dtype, device=x.device), RMS_EPS)
    if model.dtype == torch.bfloat16 and model.embedding.is_contiguous():
        out = torch.empty(hn.shape[0], model.embedding.shape[0], dtype=torch.float32, device=x.device)
        return K.linear(hn, model.embedding, out)   # tuned cuBLASLt path (csrc/forward.cu)
    return _mm(hn, model.embedding.t(), True)


def make_items(rows: list[tuple], device) -> torch.Tensor:
    """rows of (table_row, q_row0, nq, qpos0, crit_off, crit_len, dense_lo, acc_row, acc_step)."""
    arr = np.zeros((max(1, len(rows)), N.ITEM_FIELDS), dtype=np.int32)
    for i, r in enumerate(rows):
        arr[i, :9] = r
    return torch.from_numpy(arr).to(device, non_blocking=False)


# ---------------------------------------------------------------------------------
# drop-in per-request KV cache and operators
# ---------------------------------------------------------------------------------


@dataclass(frozen=True)
class KVEntry:
    """Post-rotary K/V of one token: (layers, kv_heads, head_dim) (model.py:108-119)."""

    k: torch.Tensor
    v: torch.Tensor

    def validate(self) -> None:
        k, v = torch.as_tensor(self.k), torch.as_tensor(self.v)
        if k.shape != v.shape or k.dim() != 3:
            raise ContractError("KV entry arrays must share a (layers, heads, dim) shape")
        if not (bool(torch.isfinite(k).all()) and bool(torch.isfinite(v).all())):
            raise ContractError("KV entry contains non-finite values")


class KvCache:
    """Per-request KV store (model.py:122-168) backed by a one-row device
    paged pool.  ``len`` is the committed length; slots past it hold
    provisional rows written by forwards and are never read as committed."""

    PAGE = 16

    def __init__(self, config: ModelConfig, capacity: int = 16, dtype: torch.dtype | None = None,
                 device="cuda"):
        self.config = config
        # the reference's KvCache(config, capacity) has no dtype: without one, an empty cache
        # takes the dtype of the first model that runs a forward over it (adopt_dtype)
        self._auto_dtype = dtype is None
        self.dtype = torch.float32 if dtype is None else dtype
        self.device = torch.device(device)
        self._n = 0
        self._pool = self._new_pool(max(capacity, 1))

    def _new_pool(self, capacity: int) -> PagedKvPool:
        pages = -(-capacity // self.PAGE)
        c = self.config
        pool = PagedKvPool(c.num_layers, c.num_kv_heads, c.head_dim, pages, self.PAGE, 1, pages, self.dtype,
                           self.device)
        pool.ensure_tokens(0, pages * self.PAGE)
        pool.sync_table()
        return pool

    @property
    def pool(self) -> PagedKvPool:
        return self._pool

    def adopt_dtype(self, dtype: torch.dtype) -> None:
        """Switch an empty, dtype-less cache to ``dtype`` (no-op otherwise)."""
        if self._auto_dtype and self._n == 0 and dtype != self.dtype:
            cap = self.capacity
            self.dtype = dtype
            self._pool = self._new_pool(cap)

    @property
    def capacity(self) -> int:
        return self._pool.num_pages * self.PAGE

    def __len__(self) -> int:
        return self._n

    def ensure_capacity(self, need: int) -> None:
        if need <= self.capacity:
            return
        fresh = self._new_pool(max(need, 2 * self.capacity))
        fresh.k[:, : self.capacity] = self._pool.k
        fresh.v[:, : self.capacity] = self._pool.v
        self._pool = fresh

    def append(self, entry: KVEntry) -> None:
        self.extend([entry])

    def extend(self, entries: Sequence[KVEntry]) -> None:
        if not entries:
            return
        self.ensure_capacity(self._n + len(entries))
        k = torch.stack([e.k for e in entries])
        v = torch.stack([e.v for e in entries])
        self._pool.write(0, range(self._n, self._n + len(entries)), k, v)
        self._n += len(entries)

    def truncate(self, n: int) -> None:
        if not 0 <= n <= self._n:
            raise ContractError("truncate target out of range")
        self._n = n

    def keys(self, layer: int) -> torch.Tensor:
        return self._pool.k[layer, : self._n]

    def values(self, layer: int) -> torch.Tensor:
        return self._pool.v[layer, : self._n]

    def gather(self, layer: int, positions) -> tuple[torch.Tensor, torch.Tensor]:
        idx = torch.as_tensor(np.asarray(positions, dtype=np.int64), device=self.device)
        return self._pool.k[layer, idx], self._pool.v[layer, idx]


def _check_tokens(config: ModelConfig, tokens: Sequence[int]) -> None:
    for t in tokens:
        if not 0 <= int(t) < config.vocab_size:
            raise ContractError(f"token id {t} outside vocab of {config.vocab_size}")


def _require_cache_dtype(model: ToyModel, cache: KvCache) -> None:
    cache.adopt_dtype(model.dtype)
    if cache.dtype != model.dtype:
        raise ContractError(f"cache dtype {cache.dtype} != model dtype {model.dtype}")


def forward_full(model: ToyModel, committed_kv: KvCache, new_tokens: Sequence[int], capture_scores: bool = True):
    """Verify / prefill forward (model.py:290-342).

    Returns ``(logits (n, V) fp32, [KVEntry] * n, AttentionScoreLog)``.  The
    cache's committed length is unchanged; the new tokens' K/V come back as
    entries.  The score log carries the PillarAttn accumulator
    acc[q][pos] = sum_{layer, head} exp(logit - lse) and the per-(layer, query,
    head) lse, i.e. everything importance_from_log needs (selection.py:207-218)
    without materialising logits."""
    cfg = model.config
    toks = [int(t) for t in new_tokens]
    if not toks:
        raise ContractError("forward_full needs at least one token")
    _check_tokens(cfg, toks)
    _require_cache_dtype(model, committed_kv)
    n0, n = len(committed_kv), len(toks)
    committed_kv.ensure_capacity(n0 + n)
    pool = committed_kv.pool
    dev = model.device
    shift = K.score_shift(1, cfg.num_layers, cfg.num_q_heads)
    acc = torch.zeros(n, n0 + n, dtype=torch.int64, device=dev) if capture_scores else None
    lse = torch.empty(cfg.num_layers, n, cfg.num_q_heads, dtype=torch.float32, device=dev) if capture_scores else None
    # one work item per window of ITEM_ROWS query rows (token j attends causally to [0, n0+j]):
    # every chunk is a tcgen05 verify tile on the bf16 production shapes
    step = max(1, ITEM_ROWS // cfg.group_size)
    rows = [(0, q0, min(step, n - q0), n0 + q0, 0, 0, 0, q0 if capture_scores else -1, 1)
            for q0 in range(0, n, step)]
    items = make_items(rows, dev)
    launch = AttnLaunch(items, len(rows), n0 + n, min(step, n), acc=acc, acc_row_stride=n0 + n, acc_shift=shift)
    tok = torch.tensor(toks, dtype=torch.int32, device=dev)
    rt = torch.zeros(n, dtype=torch.int32, device=dev)
    rp = torch.arange(n0, n0 + n, dtype=torch.int32, device=dev)
    q_trace = [] if capture_scores else None
    x = forward_rows(model, pool, tok, rt, rp, [launch], lse_out=lse, q_trace=q_trace)
    logits = lm_head(model, x)
    ks, vs = pool.read(0, range(n0, n0 + n))
    entries = [KVEntry(k=ks[j].clone(), v=vs[j].clone()) for j in range(n)]
    rows_fn = _score_rows_fn(model, pool, n0, n, q_trace, lse) if capture_scores else None
    log = AttentionScoreLog.from_accumulators(cfg.num_q_heads, cfg.num_kv_heads, cfg.num_layers, n0, acc, lse,
                                              acc_shift=shift, rows_fn=rows_fn,
                                              dtype_tol=1e-4 if model.dtype == torch.float32 else 2e-2)
    return logits, entries, log


def _score_rows_fn(model: ToyModel, pool: PagedKvPool, n0: int, n: int, q_trace: list, lse: torch.Tensor):
    """Deferred ScoreRow materialisation for AttentionScoreLog.layers (debug / API parity
    only): logits = q . k / sqrt(d) (+ planted bonus) in fp64 from the captured rotated
    queries and the cache's keys, rows causal as in model.py:318-334."""
    c = model.config

    def rows():
        ks, _ = pool.read(0, range(n0 + n))            # (n0 + n, L, Hkv, d)
        kd = ks.double()
        bonus = torch.zeros(n0 + n, dtype=torch.float64, device=kd.device)
        if model.planted is not None:
            pp = [p for p in model.planted.positions if p < n0 + n]
            if pp:
                bonus[torch.tensor(pp, device=kd.device)] = model.planted_bonus
        scale = 1.0 / math.sqrt(c.head_dim)
        out = []
        for l in range(c.num_layers):
            kl = kd[:, l].repeat_interleave(c.group_size, dim=1)   # (n0 + n, Hq, d)
            ql = q_trace[l].double()                             # (n, Hq, d)
            layer_rows = []
            for q in range(n):
                w = n0 + q + 1
                lg = torch.einsum("hd,jhd->hj", ql[q], kl[:w]) * scale + bonus[:w]
                layer_rows.append(ScoreRow(logits=lg, lse=lse[l, q].double()))
            out.append(layer_rows)
        return out

    return rows


def forward_sparse(model: ToyModel, committed_kv: KvCache, critical: CriticalTokenSet,
                   fresh_kv: Sequence[KVEntry], new_token: int):
    """Draft forward (model.py:345-385): the token at n0 + len(fresh) attends to
    the critical positions (< n0), every fresh entry and itself."""
    cfg = model.config
    _check_tokens(cfg, [new_token])
    _require_cache_dtype(model, committed_kv)
    n0 = len(committed_kv)
    nf = len(fresh_kv)
    pos = n0 + nf
    crit = critical.device_positions(model.device)
    if len(critical) and int(critical.positions[-1]) >= n0:
        raise ContractError("critical positions must lie inside the committed cache")
    committed_kv.ensure_capacity(pos + 1)
    pool = committed_kv.pool
    if nf:
        pool.write(0, range(n0, pos), torch.stack([e.k for e in fresh_kv]), torch.stack([e.v for e in fresh_kv]))
    dev = model.device
    items = make_items([(0, 0, 1, pos, 0, len(critical), n0, -1, 0)], dev)
    launch = AttnLaunch(items, 1, len(critical) + nf + 1, 1, crit=crit)
    tok = torch.tensor([int(new_token)], dtype=torch.int32, device=dev)
    rt = torch.zeros(1, dtype=torch.int32, device=dev)
    rp = torch.tensor([pos], dtype=torch.int32, device=dev)
    x = forward_rows(model, pool, tok, rt, rp, [launch])
    logits = lm_head(model, x)[0]
    ks, vs = pool.read(0, [pos])
    return logits, KVEntry(k=ks[0].clone(), v=vs[0].clone())


def greedy_token(logits) -> int:
    """Argmax with ties to the lowest token id (model.py:388-390), on device; fp64 rows
    (the reference's dtype) are compared in fp64."""
    t = logits if isinstance(logits, torch.Tensor) else torch.as_tensor(np.asarray(logits))
    if not t.is_cuda:
        t = t.cuda()
    if t.dtype not in (torch.float32, torch.bfloat16, torch.float64):
        t = t.double()
    t = t.reshape(1, -1).contiguous()
    out = torch.empty(1, dtype=torch.int32, device=t.device)
    K.argmax_rows(t, out)
    return int(out.item())


def greedy_tokens(logits: torch.Tensor) -> torch.Tensor:
    """Row-wise greedy_token on device (int32 [rows])."""
    out = torch.empty(logits.shape[0], dtype=torch.int32, device=logits.device)
    K.argmax_rows(logits.contiguous(), out)
    return out
