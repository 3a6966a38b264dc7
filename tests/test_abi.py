"""C-ABI library: loads, exports every symbol include/ffd.h declares, and the
host-checkable argument errors return synchronously without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ffd.h")


@pytest.fixture(scope="module")
def L():
    from paper_2404_05708_b200 import build
    build.build()
    import paper_2404_05708_b200 as ffd
    return ffd.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ffd_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    import paper_2404_05708_b200 as ffd
    names = declared_functions()
    assert set(names) == set(ffd.EXPORTED)
    for n in names:
        assert hasattr(L, n), n
    # and nm agrees (dynamic symbol table)
    out = subprocess.run(["nm", "-D", "--defined-only", ffd.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_status_strings_and_version(L):
    assert L.ffd_status_string(0) == b"ok"
    assert L.ffd_status_string(-8) == b"workspace too small"
    assert L.ffd_version() >= 100


def test_argument_errors_are_synchronous(L):
    P = ctypes.c_void_p(16)  # never dereferenced: the checks fail first
    # bad dim
    assert L.ffd_batch(P, P, P, P, 4, 5, 2, 0, P, P, 1 << 30, None) == -1
    # bad norm / dtype / int L2
    assert L.ffd_batch(P, P, P, P, 4, 2, 9, 0, P, P, 1 << 30, None) == -1
    assert L.ffd_batch(P, P, P, P, 4, 2, 2, 7, P, P, 1 << 30, None) == -1
    assert L.ffd_batch(P, P, P, P, 4, 2, 2, 1, P, P, 1 << 30, None) == -1
    # negative count, null pointers
    assert L.ffd_batch(P, P, P, P, -1, 2, 2, 0, P, P, 1 << 30, None) == -1
    assert L.ffd_batch(None, P, P, P, 4, 2, 2, 0, P, P, 1 << 30, None) == -1
    # zero pairs is a no-op
    assert L.ffd_batch(None, None, None, None, 0, 2, 2, 0, None, None, 0, None) == 0
    # workspace too small
    assert L.ffd_batch(P, P, P, P, 4, 2, 2, 0, P, P, 8, None) == -8
    # ffd_batch_maxlen: negative bounds, then the same checks as ffd_batch
    assert L.ffd_batch_maxlen(P, P, P, P, 4, -1, 4, 2, 2, 0, P, P, 1 << 30, None) == -1
    assert L.ffd_batch_maxlen(P, P, P, P, 4, 4, 4, 5, 2, 0, P, P, 1 << 30, None) == -1
    assert L.ffd_batch_maxlen(None, None, None, None, 0, 0, 0, 2, 2, 0, None, None, 0, None) == 0
    # cdist: bad shard / ld_out
    assert L.ffd_cdist(P, 10, 4, P, 10, 4, 2, 2, 0, 5, 3, P, 10, None, 0, None) == -1
    assert L.ffd_cdist(P, 10, 4, P, 10, 4, 2, 2, 0, 0, 10, P, 9, None, 0, None) == -1
    assert L.ffd_validate_batch(P, 1, P, 1, P, P, 1, 9, 0, None) == -1


def test_workspace_size_monotone(L):
    a = L.ffd_batch_workspace_bytes(10)
    b = L.ffd_batch_workspace_bytes(100000)
    assert b > a > 0
