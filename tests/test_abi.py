"""CPU-only checks of the boundary: libzk.so builds for sm_100a, loads, and exports every symbol
include/zk.h declares with the signature the binding registers (no compute calls without a GPU)."""
import os
import re
import subprocess

import pytest

from paper_2112_11880_b200 import build as zb
from paper_2112_11880_b200 import zk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDRS = [os.path.join(ROOT, "include", h) for h in ("zk.h", "zk_dist.h")]


def declared_functions():
    src = "".join(open(h).read() for h in HDRS)
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(zk_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    zb.build()
    return zk.lib()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for call in ["zk_csr_create", "zk_zcsrmv", "zk_zdotc", "zk_dznrm2", "zk_zaxpy", "zk_zscal", "zk_solve"]:
        assert call in names


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", zk.SO_PATH]).decode()
    exported = set(re.findall(r" T (zk_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert name in zk.SIGNATURES, f"binding does not register {name}"
        assert getattr(lib, name) is not None


def test_sm100a_only(lib):
    out = subprocess.check_output(["cuobjdump", "--list-elf", zk.SO_PATH]).decode()
    assert "sm_100a" in out
    for bad in ("sm_90", "sm_80", "sm_103"):
        assert bad not in out


def test_host_only_calls(lib):
    assert lib.zk_version() == 200
    assert lib.zk_status_string(-2) == b"ZK_ERR_INVALID_CSR"
    assert lib.zk_status_string(0) == b"ZK_OK"


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2112_11880_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "zk_oracle" not in txt and "liboracle" not in txt, f
    out = subprocess.check_output(["nm", "-D", zk.SO_PATH]).decode()
    assert "oracle_" not in out


def test_local_group_host_api(lib):
    """The LOCAL transport's group object is host-only: create / destroy need no GPU, bad sizes
    are rejected (zk.h: 1..16 ranks)."""
    import ctypes
    from paper_2112_11880_b200 import zk
    g = zk.LocalGroup(4)
    assert g.nranks == 4 and g.handle
    g.close()
    h = ctypes.c_void_p()
    assert lib.zk_local_group_create(ctypes.byref(h), 0) == -1
    assert lib.zk_local_group_create(ctypes.byref(h), 17) == -1
    assert lib.zk_local_group_destroy(None) == 0
