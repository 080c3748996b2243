"""CPU checks of the drop-in boundary: the C-ABI library builds, loads and exports
every entry point include/devplace_b200.h declares; the ctypes table binds them."""

import os
import re
import subprocess

import pytest

from paper_1706_04972_b200 import build as B

HEADER = os.path.join(B.ROOT, "include", "devplace_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    return B.build()


def test_header_declares_entry_points():
    names = declared()
    assert "dp_simulate_batch" in names and "dp_graph_create" in names


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dp_[a-z0-9_]+)$", out, flags=re.M))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_ctypes_table_covers_header(lib_path):
    from paper_1706_04972_b200 import _native

    L = _native.load_only()
    for n in declared():
        assert n in _native.SIGNATURES, n
        getattr(L, n)
    assert L.dp_last_error() == b""


def test_kernels_are_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_unsupported_policy_widths_raise_value_error(lib_path):
    """The reference takes any hidden/dev_dim (pkg/policy.py:127-146); this build
    implements hidden=64 and says so with a ValueError, on the host and at the C-ABI."""
    import ctypes

    from paper_1706_04972_b200 import _native
    from paper_1706_04972_b200.policy import check_policy_dims

    check_policy_dims(64, 16, 4)
    for hidden, dd, d in ((8, 16, 2), (128, 16, 2), (64, 0, 2), (64, 33, 2), (64, 16, 0), (64, 16, 33)):
        with pytest.raises(ValueError, match="this build supports"):
            check_policy_dims(hidden, dd, d)
    L = _native.load_only()
    out = ctypes.c_void_p()
    rc = L.dp_policy_create(4, 2, 8, 16, 16, 8, 64, 3, None, None, None, None, 1, ctypes.byref(out))
    # status 1 is what _native.check() turns into ValueError(message)
    assert rc == 1 and b"hidden=64" in L.dp_last_error()
