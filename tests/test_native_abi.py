"""libpd_b200.so loads on a CPU-only box and exports every symbol include/pd_b200.h declares."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_1806_03377_b200 import _native as nat

HEADER = Path(__file__).resolve().parents[1] / "include" / "pd_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(pd_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert declared() == sorted(nat.EXPORTED)


def test_library_loads_and_exports():
    if not nat.LIB_PATH.exists():
        pytest.fail("libpd_b200.so not built; run __graft_entry__.build()")
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    for sym in declared():
        assert hasattr(lib, sym), sym
    assert nat.lib().pd_abi_version() == 1


def test_struct_layouts():
    # field order of the ctypes mirrors must match the C structs (sizes on x86-64)
    assert ctypes.sizeof(nat.Epilogue) == 4 + 4 + 8 + 8 + 8 + 4 + 4 + 8 + 8 + 8 + 8 + 4 + 4 + 8 + 8 + 8 + 4 + 4 + 8
    assert ctypes.sizeof(nat.Record) == 24


def test_sass_has_tcgen05_and_tma():
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists():
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", str(nat.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA loads
    assert "LDTM" in sass  # tcgen05.ld
