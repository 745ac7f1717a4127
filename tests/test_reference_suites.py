"""Run the REFERENCE's own unit suites for the host-side drop-ins against this
package (CPU; only where /root/reference exists, i.e. the build container).

The reference's tests/test_kvpool.py and tests/test_scheduler.py import
``spardec.kvpool`` / ``spardec.scheduler`` / ``spardec.errors``; we alias those
module names to ours and execute every test function unchanged.  Nothing is
copied: the test files are read in place, read-only.
"""

import importlib.util
import inspect
import sys
import types
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
pytestmark = pytest.mark.skipif(not REF_TESTS.exists(), reason="reference checkout not present (GPU box)")


def _load_with_alias(name):
    from paper_2512_01278_b200 import errors, kvpool, scheduler

    saved = {k: sys.modules.get(k) for k in ("spardec", "spardec.kvpool", "spardec.scheduler", "spardec.errors")}
    pkg = types.ModuleType("spardec")
    pkg.__path__ = []
    sys.modules.update({"spardec": pkg, "spardec.kvpool": kvpool, "spardec.scheduler": scheduler,
                        "spardec.errors": errors})
    try:
        spec = importlib.util.spec_from_file_location(f"ref_{name}", REF_TESTS / f"{name}.py")
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v
    return mod


def _tests(mod):
    return [(n, f) for n, f in inspect.getmembers(mod, inspect.isfunction)
            if n.startswith("test_") and f.__module__ == mod.__name__]


@pytest.mark.parametrize("suite", ["test_kvpool", "test_scheduler"])
def test_reference_suite_passes_against_dropin(suite):
    mod = _load_with_alias(suite)
    tests = _tests(mod)
    assert len(tests) >= 15
    failures = []
    for name, fn in tests:
        try:
            fn()
        except Exception as e:  # noqa: BLE001 - report every failing reference test
            failures.append(f"{name}: {type(e).__name__}: {e}")
    assert not failures, "\n".join(failures)
