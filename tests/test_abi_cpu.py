"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/cmsvd.h declares; status strings; create() fails cleanly when
no GPU is visible.  No compute calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "cmsvd.h")).read()
    return sorted(set(re.findall(r"\b(cmsvd_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2601_11626_b200 import cmsvd
    L = ctypes.CDLL(cmsvd.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/cmsvd.h but not exported"
    assert set(syms) == set(cmsvd.EXPORTS)


def test_status_strings_and_version():
    from paper_2601_11626_b200 import cmsvd
    L = cmsvd.load()
    assert L.cmsvd_status_string(0) == b"CMSVD_OK"
    assert L.cmsvd_status_string(5) == b"CMSVD_E_NOCONV"
    assert b"sm_100a" in L.cmsvd_version()


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2601_11626_b200 import Context, CmsvdError
    with pytest.raises(CmsvdError):
        Context(0)


def test_sm100a_code_in_library():
    """The library holds sm_100a SASS (cuobjdump lists the arch)."""
    import subprocess
    from paper_2601_11626_b200 import cmsvd
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", cmsvd.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
