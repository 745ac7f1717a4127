"""Typed Python entry points over the C ABI (one call = one stream-ordered
launch on the current CUDA stream).  Shapes are validated here, mirroring the
reference's host-side contract checks, before anything is launched."""

from __future__ import annotations

import ctypes
import math

import torch

from . import _native as N
from .errors import ContractError


def rope_kv_write(qkv: torch.Tensor, row_table: torch.Tensor, row_pos: torch.Tensor, pool, layer: int,
                  q_heads: int, q_out: torch.Tensor) -> None:
    """K5: RoPE q/k at row_pos, write k/v into the paged pool, rotated q to q_out."""
    rows = qkv.shape[0]
    if rows == 0:
        return
    N.require_cuda(qkv, "qkv")
    if qkv.stride(1) != 1 or q_out.dtype != pool.dtype or qkv.dtype != pool.dtype:
        raise ContractError("rope_kv_write: qkv/q_out must match the pool dtype with unit inner stride")
    desc = pool.desc()
    N.check(N.lib().sd_rope_kv_write(qkv.data_ptr(), qkv.stride(0), rows, row_table.data_ptr(),
                                     row_pos.data_ptr(), ctypes.byref(desc), layer, q_heads,
                                     q_out.data_ptr(), N.stream_handle()), "sd_rope_kv_write")


_WS: dict = {}
_NEED: list = [None, 0]  # last (descriptor, launch shape) -> workspace bytes


def _zeroed_workspace(nbytes: int, device) -> torch.Tensor:
    """Per-device attention workspace: zero-filled when allocated, and every
    sd_attention call hands it back zero-filled (spardec_b200.h), so it is reused."""
    key = torch.device(device)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=key)
        _WS[key] = ws
    return ws


def score_shift(rows_per_entry: int, layers: int, q_heads: int) -> int:
    """Fixed-point scale 2^shift of the score accumulators: the largest possible entry
    (rows summed into it x layers x q heads, each probability <= 1) stays below 2^62."""
    worst = max(1, int(rows_per_entry) * int(layers) * int(q_heads))
    return max(0, min(62, 62 - math.ceil(math.log2(worst))))


def scores_to_float(acc: torch.Tensor, shift: int) -> torch.Tensor:
    """Fixed-point accumulators -> fp64 values (exact up to 2^53 units)."""
    return acc.double() * (2.0 ** -shift)


def attention(q: torch.Tensor, out: torch.Tensor, pool, layer: int, items: torch.Tensor, num_items: int,
              max_keys: int, max_nq: int, q_heads: int, *, crit: torch.Tensor | None = None,
              lse: torch.Tensor | None = None, acc: torch.Tensor | None = None, acc_row_stride: int = 0,
              acc_shift: int = 0, planted: torch.Tensor | None = None, planted_bonus: float = 0.0,
              scale: float | None = None, workspace: torch.Tensor | None = None,
              force_generic: bool = False) -> None:
    """K1/K2: paged GQA attention over the work items (see spardec_b200.h).  ``acc`` is an
    int64 tensor of fixed-point score accumulators (unit 2^-acc_shift)."""
    if num_items == 0:
        return
    if acc is not None and acc.dtype != torch.int64:
        raise ContractError("attention: score accumulators are int64 fixed point (see score_shift)")
    desc = pool.desc()
    lib = N.lib()
    key = (desc.kv_heads, desc.head_dim, desc.dtype, num_items, max_keys, max_nq, q_heads)
    if key == _NEED[0]:  # every layer of one iteration asks the same question
        need = _NEED[1]
    else:
        need = lib.sd_attention_workspace_bytes(num_items, max_keys, max_nq, q_heads, ctypes.byref(desc))
        _NEED[0], _NEED[1] = key, need
    if force_generic:
        G = q_heads // pool.kv_heads
        need = num_items * pool.kv_heads * (max_nq * G * max_keys + 3 * max_keys) * 4
    if need > 0 and (workspace is None or workspace.numel() * workspace.element_size() < need):
        workspace = _zeroed_workspace(need, q.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    if scale is None:
        scale = 1.0 / (pool.head_dim ** 0.5)
    n_planted = 0 if planted is None else planted.numel()
    N.check(lib.sd_attention(q.data_ptr(), out.data_ptr(), N.ptr(lse), ctypes.byref(desc), layer,
                             items.data_ptr(), num_items, max_keys, max_nq, N.ptr(crit), N.ptr(acc),
                             acc_row_stride, acc_shift, N.ptr(planted), n_planted, planted_bonus, q_heads, scale,
                             N.ptr(workspace), ws_bytes, 1 if force_generic else 0, N.stream_handle()),
            "sd_attention")


def attention_pair(q: torch.Tensor, out: torch.Tensor, pool, layer: int, verify: dict, draft: dict, q_heads: int,
                   *, planted: torch.Tensor | None = None, planted_bonus: float = 0.0,
                   scale: float | None = None) -> bool:
    """f3: a layer's verify launch (dense items; keys items / num_items / max_keys / max_nq /
    acc / acc_row_stride / acc_shift) and draft launch (items / num_items / max_keys / crit) in
    ONE launch.  Returns False (nothing launched) when the pair does not qualify."""
    def desc(d):
        return N.AttnLaunchDesc(d["items"].data_ptr(), d["num_items"], d["max_keys"], d.get("max_nq", 1),
                                d.get("acc_shift", 0), N.ptr(d.get("crit")), N.ptr(d.get("acc")),
                                d.get("acc_row_stride", 0))
    dv, dd = desc(verify), desc(draft)
    if scale is None:
        scale = 1.0 / (pool.head_dim ** 0.5)
    n_planted = 0 if planted is None else planted.numel()
    pdesc = pool.desc()
    rc = N.lib().sd_attention_pair(q.data_ptr(), out.data_ptr(), ctypes.byref(pdesc), layer, ctypes.byref(dv),
                                   ctypes.byref(dd), N.ptr(planted), n_planted, planted_bonus, q_heads, scale,
                                   N.stream_handle())
    if rc == 1:
        return False
    N.check(rc, "sd_attention_pair")
    return True


def select_critical(acc: torch.Tensor, acc_req_stride: int, acc_row_stride: int, acc_shift: int,
                    n_rows: torch.Tensor, kv_len: torch.Tensor, sparsity: float, num: int,
                    importance: torch.Tensor, crit: torch.Tensor, crit_len: torch.Tensor,
                    budget: torch.Tensor | None = None, req_index: torch.Tensor | None = None) -> None:
    """K3: importance (fp64) = sum of the surviving fixed-point score rows; budget; tie-exact
    top-k.  ``req_index[r]`` (optional) redirects request r to row req_index[r] of
    acc / importance / crit / crit_len / budget."""
    if num == 0:
        return
    if acc.dtype != torch.int64 or importance.dtype != torch.float64:
        raise ContractError("select_critical: int64 accumulators and float64 importance expected")
    N.check(N.lib().sd_select_critical(acc.data_ptr(), acc_req_stride, acc_row_stride, acc_shift, n_rows.data_ptr(),
                                       kv_len.data_ptr(), float(sparsity), num, N.ptr(req_index),
                                       importance.data_ptr(),
                                       importance.stride(0), crit.data_ptr(), crit.stride(0),
                                       crit_len.data_ptr(), N.ptr(budget), N.stream_handle()),
            "sd_select_critical")


def topk(values: torch.Tensor, n: torch.Tensor, budget: torch.Tensor, out: torch.Tensor,
         out_len: torch.Tensor) -> None:
    """Batched tie-exact top-k over rows of float32/float64 values."""
    if values.dtype == torch.float32:
        code = 0
    elif values.dtype == torch.float64:
        code = 2
    else:
        raise ContractError("topk values must be float32 or float64")
    N.check(N.lib().sd_topk(values.data_ptr(), code, values.stride(0), n.data_ptr(), budget.data_ptr(),
                            values.shape[0], out.data_ptr(), out.stride(0), out_len.data_ptr(),
                            N.stream_handle()), "sd_topk")


def argmax_rows(logits: torch.Tensor, out: torch.Tensor) -> None:
    """K4a: per-row argmax with ties to the lowest id."""
    rows, vocab = logits.shape
    if logits.stride(1) != 1:
        raise ContractError("argmax_rows: logits rows must be contiguous")
    N.check(N.lib().sd_argmax_rows(logits.data_ptr(), N.dtype_code(logits.dtype), logits.stride(0), rows,
                                   vocab, out.data_ptr(), N.stream_handle()), "sd_argmax_rows")


def greedy_accept(targets: torch.Tensor, tokens: torch.Tensor, row0: torch.Tensor, nrows: torch.Tensor,
                  accepted: torch.Tensor, bonus: torch.Tensor) -> None:
    """K4b: longest accepted draft prefix and the bonus token per verify member."""
    N.check(N.lib().sd_greedy_accept(targets.data_ptr(), tokens.data_ptr(), row0.data_ptr(), nrows.data_ptr(),
                                     row0.numel(), accepted.data_ptr(), bonus.data_ptr(), N.stream_handle()),
            "sd_greedy_accept")


def step_prepare(plan: torch.Tensor, n_members: int, k: int, crit_cap: int, n_kv: torch.Tensor,
                 last_tok: torch.Tensor, drafted: torch.Tensor, crit_len: torch.Tensor, tokens: torch.Tensor,
                 row_table: torch.Tensor, row_pos: torch.Tensor, v_items: torch.Tensor, d_items: torch.Tensor,
                 acc: torch.Tensor, acc_row_stride: int) -> None:
    """Iteration inputs (tokens, positions, work items) from the device-resident request state."""
    N.check(N.lib().sd_step_prepare(plan.data_ptr(), n_members, k, crit_cap, n_kv.data_ptr(), last_tok.data_ptr(),
                                    drafted.data_ptr(), crit_len.data_ptr(), tokens.data_ptr(), row_table.data_ptr(),
                                    row_pos.data_ptr(), v_items.data_ptr(), d_items.data_ptr(), acc.data_ptr(),
                                    acc_row_stride, N.stream_handle()), "sd_step_prepare")


def step_commit(plan: torch.Tensor, n_members: int, k: int, targets: torch.Tensor, n_kv: torch.Tensor,
                last_tok: torch.Tensor, drafted: torch.Tensor, sel_rows: torch.Tensor, sel_kv: torch.Tensor,
                sel_slot: torch.Tensor, results: torch.Tensor) -> None:
    """Drafts record their token; verifies accept / roll back on the device (engine.py:231-240)."""
    N.check(N.lib().sd_step_commit(plan.data_ptr(), n_members, k, targets.data_ptr(), n_kv.data_ptr(),
                                   last_tok.data_ptr(), drafted.data_ptr(), sel_rows.data_ptr(), sel_kv.data_ptr(),
                                   sel_slot.data_ptr(), results.data_ptr(), N.stream_handle()), "sd_step_commit")


def rmsnorm_cast(x: torch.Tensor, out: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    """Glue: RMSNorm without gain of fp32 rows, cast to out.dtype (one launch)."""
    if x.dtype != torch.float32 or not x.is_contiguous() or not out.is_contiguous():
        raise ContractError("rmsnorm_cast: x must be contiguous fp32")
    N.check(N.lib().sd_rmsnorm_cast(x.data_ptr(), x.shape[0], x.shape[1], eps, out.data_ptr(),
                                    N.dtype_code(out.dtype), N.stream_handle()), "sd_rmsnorm_cast")
    return out


def linear(a: torch.Tensor, w: torch.Tensor, out: torch.Tensor, accumulate: bool = False) -> torch.Tensor:
    """out (+)= a . w^T on the library's tuned cuBLASLt path (a, w bf16 contiguous, w [N][K];
    out fp32 or bf16 [R][N])."""
    if a.dtype != torch.bfloat16 or w.dtype != torch.bfloat16 or not (a.is_contiguous() and w.is_contiguous()
                                                                      and out.is_contiguous()):
        raise ContractError("linear: contiguous bf16 a and w required")
    R, Kd = a.shape
    if w.shape[1] != Kd or tuple(out.shape) != (R, w.shape[0]):
        raise ContractError("linear: shape mismatch")
    N.check(N.lib().sd_linear(a.data_ptr(), w.data_ptr(), out.data_ptr(), R, w.shape[0], Kd,
                              1 if out.dtype == torch.float32 else 0, 1.0 if accumulate else 0.0,
                              N.stream_handle()), "sd_linear")
    return out


def launch_count() -> int:
    return int(N.lib().sd_launch_count())
