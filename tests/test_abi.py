"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/ltlgrid_gpu.h declares, is built for sm_100a, and its host-only
validator reproduces the reference's messages."""
import ctypes as C
import json
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, has_gpu
from paper_1810_02612_b200 import _native as N

HEADER = os.path.join(ROOT, "include", "ltlgrid_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ltlg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_python_binds():
    assert declared_functions() == sorted(N.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = N.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", N.GPU_SO], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ltlg_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert getattr(L, name) is not None
    assert L.ltlg_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", N.GPU_SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_cpu_fallback_without_device():
    if has_gpu():
        pytest.skip("a GPU is present")
    from paper_1810_02612_b200 import LabelEngine, LtlgError

    with pytest.raises(LtlgError, match="no CUDA device"):
        LabelEngine()


def test_host_validator_matches_reference_messages():
    L = N.lib()
    with open(os.path.join(GOLDEN, "validate.json")) as f:
        cases = json.load(f)
    for c in cases:
        off = np.array(c["offsets"], np.uint64)
        idx = np.array(c["indices"], np.uint32)
        buf = C.create_string_buffer(256)
        st = L.ltlg_validate_csr(c["rows"], c["cols"], off.ctypes.data, off.size, idx.ctypes.data, idx.size, buf, 256)
        if c["error"] is None:
            assert st == N.LTLG_OK, c
        else:
            assert st == N.LTLG_EINVAL and buf.value.decode() == c["error"], c
    off = np.array([0, 1, 3], np.uint64)
    idx = np.array([4, 1, 2], np.uint32)
    buf = C.create_string_buffer(256)
    assert L.ltlg_validate_csr(2, 5, off.ctypes.data, 3, idx.ctypes.data, 3, buf, 256) == N.LTLG_OK
