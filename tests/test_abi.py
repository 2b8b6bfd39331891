"""CPU-side checks of the C-ABI boundary: the library builds, loads without a GPU,
exports every symbol include/*.h declares, and rejects host-checkable bad arguments
before touching the device."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2506_01979_b200 import _lib
    from paper_2506_01979_b200.build import build

    build()
    return _lib


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", src))
    return names


def test_every_declared_symbol_is_exported(L):
    lib = L.lib()
    decl = declared_symbols()
    assert {"sb_verify_branches", "sb_select_branch", "sb_draft_confidence"} <= decl
    for n in decl:
        assert hasattr(lib, n), n
    assert set(L.EXPORTS) == decl


def test_version_and_status_strings(L):
    lib = L.lib()
    assert b"sm_100a" in lib.sb_version()
    assert lib.sb_status_string(L.SB_ERR_WORKSPACE) == b"workspace too small"


def _dims(L, **kw):
    d = dict(B=4, K=2, G=8, V=1000, v_offset=0, v_total=1000, row_stride=1000, seq_stride=0,
             dtype=L.SB_BF16, reserved=0)
    d.update(kw)
    return L.sb_dims(**d)


def test_workspace_bytes(L):
    lib = L.lib()
    n = lib.sb_workspace_bytes(ctypes.byref(_dims(L)))
    assert n > 0 and n % 256 == 0
    n2 = lib.sb_workspace_bytes(ctypes.byref(_dims(L, B=2048)))
    assert n2 > n
    for bad in (dict(B=0), dict(K=0), dict(K=33), dict(G=32), dict(G=-1), dict(V=1),
                dict(row_stride=999), dict(dtype=7), dict(reserved=1), dict(v_offset=5)):
        assert lib.sb_workspace_bytes(ctypes.byref(_dims(L, **bad))) == 0, bad


def test_invalid_args_rejected_on_host(L):
    lib = L.lib()
    d = _dims(L)
    nul = [None] * 18
    rc = lib.sb_verify_branches(ctypes.byref(d), *nul, 0, None)
    assert rc == L.SB_ERR_INVALID_ARG
    rc = lib.sb_select_branch(ctypes.byref(d), *[None] * 8, 0, *[None] * 14, 0, None)
    assert rc == L.SB_ERR_INVALID_ARG
    rc = lib.sb_draft_confidence(ctypes.byref(d), None, None, 0, 0.2, 1.0, 6, *[None] * 10, 0, None)
    assert rc == L.SB_ERR_INVALID_ARG
    # a workspace too small is reported before any launch (fake non-null pointers)
    fake = ctypes.c_void_p(256)
    args = [fake] * 18
    args[16] = None  # comm
    rc = lib.sb_verify_branches(ctypes.byref(d), *args, 16, None)
    assert rc == L.SB_ERR_WORKSPACE
    # bad confidence parameters
    rc = lib.sb_draft_confidence(ctypes.byref(d), fake, None, 0, 1.5, 1.0, 6, *[fake] * 8, None,
                                 fake, 1 << 30, None)
    assert rc == L.SB_ERR_INVALID_ARG


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_2506_01979_b200 import _lib

    monkeypatch.setattr(_lib, "SO", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()


def test_product_path_never_imports_oracle():
    """The CUDA path and the oracle share no code."""
    pkg = os.path.join(ROOT, "paper_2506_01979_b200")
    pat = re.compile(r"import\s+oracle|from\s+oracle|liboracle|oracle\.h|oracle/")
    for f in glob.glob(os.path.join(pkg, "**", "*.*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".h")):
            assert not pat.search(open(f).read()), f


def test_invalid_args_rejected_on_host_next_rows(L):
    """The §8.6 entry points and the reuse variant check their arguments before any
    launch (fake non-null device pointers never get dereferenced)."""
    lib = L.lib()
    d = _dims(L)
    fake = ctypes.c_void_p(256)
    # sb_verify_branches_reuse: a conf workspace is required
    args = [fake] * 16 + [None, fake]
    assert lib.sb_verify_branches_reuse(ctypes.byref(d), *args, 1 << 30, None) == L.SB_ERR_INVALID_ARG
    # sb_spawn_branches: k_max in [1, 16]
    assert lib.sb_spawn_branches(ctypes.byref(d), fake, None, None, 0, 17, fake, fake, None, None,
                                 None) == L.SB_ERR_INVALID_ARG
    # sb_kv_rollback: rows must be 16-byte multiples
    assert lib.sb_kv_rollback(4, 2, 3, fake, 24, 32, fake, None, None) == L.SB_ERR_INVALID_ARG
    assert lib.sb_kv_rollback(4, 2, 3, fake, 32, 32, None, None, None) == L.SB_ERR_INVALID_ARG  # keep_mask
    # sb_tree_verify: K must be 1
    assert lib.sb_tree_workspace_bytes(ctypes.byref(d)) == 0  # d has K = 4
    assert lib.sb_tree_verify(ctypes.byref(d), *[fake] * 15, fake, 1 << 30, None) == L.SB_ERR_INVALID_ARG
    # sb_hrad_predict: B >= 1, Dz a multiple of 64 (12 tensors, workspace, bytes, stream)
    hr = [fake] * 12 + [fake, 1 << 30, None]
    assert lib.sb_hrad_predict(0, 256, 8, *hr) == L.SB_ERR_INVALID_ARG
    assert lib.sb_hrad_predict(4, 200, 8, *hr) == L.SB_ERR_UNSUPPORTED
    assert lib.sb_hrad_predict(4, 256, 40, *hr) == L.SB_ERR_INVALID_ARG  # G > 31
