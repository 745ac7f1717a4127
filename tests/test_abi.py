"""C-ABI library checks that need no GPU: it loads, exports every symbol the
header declares, and reports its ABI version."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    src = (ROOT / "include" / "spardec_b200.h").read_text()
    return sorted(set(re.findall(r"\b(sd_[a-z_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("sd_attention", "sd_rope_kv_write", "sd_select_critical", "sd_topk", "sd_argmax_rows",
                 "sd_greedy_accept", "sd_last_error", "sd_abi_version"):
        assert must in names


def test_library_loads_and_exports_every_symbol():
    from paper_2512_01278_b200 import _native as N
    lib = N.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(N.SIGNATURES)
    assert lib.sd_abi_version() == N.ABI_VERSION == 2
    assert lib.sd_build_id().decode() == N.source_build_id()  # built from these sources
    assert lib.sd_last_error() == b""


def test_contract_violation_maps_to_contract_error():
    import ctypes
    from paper_2512_01278_b200 import _native as N
    from paper_2512_01278_b200.errors import ContractError
    lib = N.load_library()
    rc = lib.sd_select_critical(None, 0, 0, 0, None, None, 0.5, 1, None, None, 0, None, 0, None, None, None)
    assert rc < 0
    with pytest.raises(ContractError, match="null pointer"):
        N.check(rc, "sd_select_critical")
    rc = lib.sd_topk(None, 7, 0, None, None, 1, None, 0, None, None)
    assert rc < 0 and b"float32" in lib.sd_last_error()
