"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a, loads,
and exports every function include/sparsesync.h declares (no compute calls —
there is no GPU here). Also: the product package never imports the oracle."""
import ast
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sparsesync.h")
PEER_HEADER = os.path.join(ROOT, "include", "sparsesync_peer.h")
PKG = os.path.join(ROOT, "paper_2605_07330_b200")


def declared(path=HEADER):
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sync_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_07330_b200 import build
    build.build()
    import paper_2605_07330_b200 as ss
    return ss.lib()


def test_header_declares_the_boundary():
    names = declared()
    for required in ["sync_extract", "sync_extract_batched", "sync_compress", "sync_decompress", "sync_bucket_pack",
                     "sync_bucket_unpack", "sync_apply", "sync_commit_snapshot", "sync_decompress_apply"]:
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    import paper_2605_07330_b200 as ss
    assert sorted(ss.EXPORTS) == declared()


def test_library_exports_peer_plumbing(lib):
    """include/sparsesync_peer.h (NVLink peer-memory transfer plumbing) is exported too."""
    import paper_2605_07330_b200 as ss
    names = declared(PEER_HEADER)
    assert names and not [n for n in names if not hasattr(lib, n)]
    assert sorted(ss.PEER_EXPORTS) == names


def test_library_is_sm100a_sass(lib):
    import paper_2605_07330_b200 as ss
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ss.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_strerror_host_only(lib):
    import paper_2605_07330_b200 as ss
    assert ss.strerror(ss.SYNC_ERR_CRC) == "CRC-32 mismatch"
    assert ss.strerror(0) == "ok"


def test_host_side_argument_errors(lib):
    import ctypes
    import paper_2605_07330_b200 as ss
    # bad manifest: numel >= 2^31 is rejected without touching a device
    arr = (ctypes.c_uint64 * 1)(1 << 31)
    m = ss._Manifest(1, arr)
    c = ss._Config(1 << 20, 100, 1, 0)
    need = ctypes.c_size_t()
    assert lib.sync_workspace_size(ctypes.byref(m), ctypes.byref(c), ctypes.byref(need)) == ss.SYNC_ERR_ARG
    arr[0] = 1000
    assert lib.sync_workspace_size(ctypes.byref(m), ctypes.byref(c), ctypes.byref(need)) == ss.SYNC_OK
    assert need.value > 0
    c.bucket_limit = 8
    assert lib.sync_workspace_size(ctypes.byref(m), ctypes.byref(c), ctypes.byref(need)) == ss.SYNC_ERR_ARG
    c.bucket_limit = 1 << 20
    for dt, want in ((0, ss.SYNC_OK), (ss.SYNC_DTYPE_BF16, ss.SYNC_OK), (ss.SYNC_DTYPE_FP16, ss.SYNC_OK),
                     (ss.SYNC_DTYPE_FP8, ss.SYNC_OK), (4, ss.SYNC_ERR_DTYPE)):
        c.dtype = dt
        assert lib.sync_workspace_size(ctypes.byref(m), ctypes.byref(c), ctypes.byref(need)) == want


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), f
            if f.endswith((".cu", ".cuh", ".h")):
                assert "oracle" not in open(os.path.join(dirpath, f)).read().replace("oracle/", ""), f
