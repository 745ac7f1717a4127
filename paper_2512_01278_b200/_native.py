"""ctypes binding of the in-tree C-ABI library ``_lib/libspardec_b200.so``.

There is no CPU fallback: if the library is missing or no CUDA device is
present, every kernel entry point raises.  Declarations mirror
``include/spardec_b200.h`` one to one.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

from .errors import ContractError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libspardec_b200.so"

SD_DTYPE_F32 = 0
SD_DTYPE_BF16 = 1
ITEM_FIELDS = 12
PLAN_FIELDS = 6   # SD_PLAN_FIELDS
PLAN_DRAFT, PLAN_VERIFY = 0, 1
(F_TABLE_ROW, F_Q_ROW0, F_NQ, F_QPOS0, F_CRIT_OFF, F_CRIT_LEN, F_DENSE_LO, F_ACC_ROW, F_ACC_STEP) = range(9)

_c_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64


class PagedKvDesc(ctypes.Structure):
    _fields_ = [
        ("k", _c_p), ("v", _c_p), ("layer_stride", _i64), ("num_slots", _i64),
        ("block_table", _c_p), ("table_stride", _i32), ("page_shift", _i32),
        ("kv_heads", _i32), ("head_dim", _i32), ("dtype", _i32), ("reserved", _i32),
    ]


# name -> (restype, argtypes); must match include/spardec_b200.h
class LayerWeights(ctypes.Structure):
    _fields_ = [("w_qkv", ctypes.c_void_p), ("wo", ctypes.c_void_p), ("mlp_in", ctypes.c_void_p),
                ("mlp_out", ctypes.c_void_p)]


class AttnLaunchDesc(ctypes.Structure):
    _fields_ = [("items", ctypes.c_void_p), ("num_items", ctypes.c_int32), ("max_keys", ctypes.c_int32),
                ("max_nq", ctypes.c_int32), ("acc_shift", ctypes.c_int32), ("crit", ctypes.c_void_p),
                ("acc", ctypes.c_void_p), ("acc_row_stride", ctypes.c_int64)]


SIGNATURES = {
    "sd_abi_version": (_i32, []),
    "sd_build_id": (ctypes.c_char_p, []),
    "sd_last_error": (ctypes.c_char_p, []),
    "sd_launch_count": (_i64, []),
    "sd_rope_kv_write": (ctypes.c_int, [_c_p, _i64, _i32, _c_p, _c_p, ctypes.POINTER(PagedKvDesc), _i32, _i32,
                                        _c_p, _c_p]),
    "sd_attention_workspace_bytes": (_i64, [_i32, _i32, _i32, _i32, ctypes.POINTER(PagedKvDesc)]),
    "sd_attention": (ctypes.c_int, [_c_p, _c_p, _c_p, ctypes.POINTER(PagedKvDesc), _i32, _c_p, _i32, _i32, _i32,
                                    _c_p, _c_p, _i64, _i32, _c_p, _i32, ctypes.c_float, _i32, ctypes.c_float,
                                    _c_p, _i64, _i32, _c_p]),
    "sd_select_critical": (ctypes.c_int, [_c_p, _i64, _i64, _i32, _c_p, _c_p, ctypes.c_double, _i32, _c_p, _c_p,
                                          _i64, _c_p, _i64, _c_p, _c_p, _c_p]),
    "sd_topk": (ctypes.c_int, [_c_p, _i32, _i64, _c_p, _c_p, _i32, _c_p, _i64, _c_p, _c_p]),
    "sd_argmax_rows": (ctypes.c_int, [_c_p, _i32, _i64, _i32, _i32, _c_p, _c_p]),
    "sd_greedy_accept": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _i32, _c_p, _c_p, _c_p]),
    "sd_forward_workspace_bytes": (ctypes.c_int64, [_i32, _i32, ctypes.c_int64]),
    "sd_linear": (ctypes.c_int, [_c_p, _c_p, _c_p, _i32, _i32, _i32, _i32, ctypes.c_float, _c_p]),
    "sd_attention_pair": (ctypes.c_int, [_c_p, _c_p, ctypes.POINTER(PagedKvDesc), _i32, ctypes.POINTER(AttnLaunchDesc),
                                         ctypes.POINTER(AttnLaunchDesc), _c_p, _i32, ctypes.c_float, _i32,
                                         ctypes.c_float, _c_p]),
    "sd_step_prepare": (ctypes.c_int, [_c_p, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                                       _c_p, ctypes.c_int64, _c_p]),
    "sd_step_commit": (ctypes.c_int, [_c_p, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "sd_rmsnorm_cast": (ctypes.c_int, [_c_p, _i32, _i32, ctypes.c_float, _c_p, _i32, _c_p]),
    "sd_forward_graph_stats": (_i64, [_i32]),
    "sd_forward_layers": (ctypes.c_int, [ctypes.POINTER(LayerWeights), _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                                         _i32, _i32, _i32, _c_p, _c_p, ctypes.POINTER(PagedKvDesc),
                                         ctypes.POINTER(AttnLaunchDesc), _i32, _c_p, _i32, ctypes.c_float,
                                         ctypes.c_float, ctypes.c_float, _c_p, _i64, _c_p, _i32, _c_p]),
}

_LIB = None
ABI_VERSION = 2


def source_build_id() -> str | None:
    """Hash of the CUDA sources + flags the library must have been built from (compiled into
    the library as sd_build_id()); None when the sources are not shipped."""
    try:
        from .csrc import build as B
    except ImportError:  # pragma: no cover
        return None
    return B.source_stamp()


def load_library(path: Path | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = Path(path or os.environ.get("SPARDEC_B200_LIB", LIB_PATH))
    if not p.exists():
        raise ImportError(
            f"libspardec_b200.so not found at {p}; build it with "
            "`python -m paper_2512_01278_b200.csrc.build` (there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        try:
            fn = getattr(lib, name)
        except AttributeError as e:
            raise ImportError(f"{p} is stale (missing {name}); rebuild it") from e
        fn.restype = res
        fn.argtypes = args
    if lib.sd_abi_version() != ABI_VERSION:
        raise ImportError("libspardec_b200.so ABI version mismatch")
    want = source_build_id()
    have = lib.sd_build_id().decode()
    if want is not None and have != want:
        raise ImportError(f"{p} was built from other sources (build id {have[:12]} != {want[:12]}); "
                          "rebuild it with `python -m paper_2512_01278_b200.csrc.build`")
    _LIB = lib
    return lib


def lib() -> ctypes.CDLL:
    return load_library()


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = lib().sd_last_error().decode(errors="replace")
    if rc < 0:
        raise ContractError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA error {rc}: {msg}")


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


SD_DTYPE_F64 = 2


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return SD_DTYPE_F32
    if dt == torch.float64:
        return SD_DTYPE_F64
    if dt == torch.bfloat16:
        return SD_DTYPE_BF16
    raise ContractError(f"unsupported dtype {dt}")


def require_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise ContractError(f"{name} must be a CUDA tensor (no CPU fallback)")
