"""C-ABI library: loads without a GPU and exports every symbol include/runsort_b200.h declares."""
import ctypes
import os
import re

import pytest

from paper_1805_04154_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    with open(os.path.join(REPO, "include", "runsort_b200.h")) as fh:
        src = fh.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTS) == declared_functions()


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value


def test_pure_host_queries():
    L = _lib.lib()
    assert L.rs_version() >= 100
    assert L.rs_max_min_run_len(_lib.RS_KEY_I32, 0) >= 1024
    assert L.rs_max_min_run_len(_lib.RS_KEY_I64, 8) >= 1024
    small = L.rs_workspace_bytes(0, _lib.RS_KEY_I32, 0, 1000, 24)
    big = L.rs_workspace_bytes(0, _lib.RS_KEY_I32, 0, 10**7, 24)
    assert 0 < small < big
    # scratch buffer dominates: about one key array plus O(n/w) metadata
    assert 4 * 10**7 <= big <= 4 * 10**7 * 4


def test_status_codes_map_to_reference_exceptions():
    for rc, exc in ((_lib.RS_EINVAL, ValueError), (_lib.RS_EINVARIANT, AssertionError),
                    (_lib.RS_ENOMEM, MemoryError), (_lib.RS_EUNSUPPORTED, NotImplementedError),
                    (_lib.RS_ECUDA, RuntimeError)):
        with pytest.raises(exc):
            _lib.check(rc)
    _lib.check(_lib.RS_OK)


def test_invalid_arguments_rejected_before_any_device_work():
    L = _lib.lib()
    out = _lib.RsMetrics()
    assert L.rs_sort(0, _lib.RS_KEY_I32, None, 0, None, 10, 0, 0, None, 0, None, ctypes.byref(out), None) == _lib.RS_EINVAL
    assert L.rs_sort(0, _lib.RS_KEY_I32, None, 0, None, 10, 24, 7, None, 0, None, ctypes.byref(out), None) == _lib.RS_EINVAL
    assert L.rs_sort(0, 9, None, 0, None, 10, 24, 0, None, 0, None, ctypes.byref(out), None) == _lib.RS_EUNSUPPORTED
    assert L.rs_sort(0, _lib.RS_KEY_I32, None, 3, None, 10, 24, 0, None, 0, None, ctypes.byref(out), None) == _lib.RS_EUNSUPPORTED
    # n <= 1 returns immediately (reference sorters.py:445-450)
    assert L.rs_sort(0, _lib.RS_KEY_I32, None, 0, None, 1, 24, 0, None, 0, None, ctypes.byref(out), None) == _lib.RS_OK
    assert out.runs_detected == 1 and out.merge_cost == 0


def test_peeksort_workspace_is_compact_by_default():
    """Peeksort's default workspace stays within 2x powersort's;
    RS_ALGO_FULL_WS sizes the replay arrays for n + 1 recursive calls."""
    L = _lib.lib()
    for kc, tb in ((_lib.RS_KEY_I32, 0), (_lib.RS_KEY_I32, 4), (_lib.RS_KEY_I64, 0), (_lib.RS_KEY_I64, 8)):
        for n in (10**7, 10**8):
            power = L.rs_workspace_bytes(_lib.RS_ALGO_POWERSORT, kc, tb, n, 24)
            peek = L.rs_workspace_bytes(_lib.RS_ALGO_PEEKSORT, kc, tb, n, 24)
            full = L.rs_workspace_bytes(_lib.RS_ALGO_PEEKSORT | _lib.RS_ALGO_FULL_WS, kc, tb, n, 24)
            assert peek <= 2 * power, (kc, tb, n, peek / n, power / n)
            assert full > 5 * peek
    # small n: the compact capacity already is n + 1
    assert L.rs_workspace_bytes(_lib.RS_ALGO_PEEKSORT, _lib.RS_KEY_I32, 0, 3000, 24) == \
        L.rs_workspace_bytes(_lib.RS_ALGO_PEEKSORT | _lib.RS_ALGO_FULL_WS, _lib.RS_KEY_I32, 0, 3000, 24)
    # the flag means nothing to the other algorithms
    assert L.rs_workspace_bytes(_lib.RS_ALGO_POWERSORT | _lib.RS_ALGO_FULL_WS, _lib.RS_KEY_I32, 0, 10**6, 24) == \
        L.rs_workspace_bytes(_lib.RS_ALGO_POWERSORT, _lib.RS_KEY_I32, 0, 10**6, 24)
