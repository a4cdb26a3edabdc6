"""CPU: the C-ABI library builds for sm_100a, loads, and exports every entry
point include/diffmpm.h declares (no compute without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "diffmpm.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dm_[a-z_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2412_12089_b200 import build
    so = build.build()
    lib = ctypes.CDLL(so)
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_library_is_sm100a():
    from paper_2412_12089_b200 import build
    so = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    """Without a device the API raises instead of falling back to a CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2412_12089_b200 import api
    sim = {"dims": (16, 16, 16), "dx": 1 / 16, "dt": 1e-4}
    with pytest.raises(RuntimeError):
        api.MpmBatch(sim, [{"kind": "fluid", "volume": 1e-6}], [], 1, 8, 1, 1)
