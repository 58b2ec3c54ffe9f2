"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/gsf_cuda.h
declares, fails loudly (no CPU fallback) without a device, and its host-only pieces work."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2403_16095_b200 import abi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gsf_cuda.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(gsf_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = abi.load()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
        assert n in abi.SIGNATURES, f"{n} missing from the ctypes signature table"
    assert lib.gsf_abi_version() == 1


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {abi.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is visible")
    with pytest.raises(abi.GsfError):
        api.Context(0)


def test_ba_partition_covers_window_once():
    for n in (1, 3, 16):
        for world in (1, 2, 4, 8):
            owned = np.stack([api.ba_partition(n, world, r) for r in range(world)])
            assert (owned.sum(0) == 1).all()
            for r in range(world):
                assert list(np.nonzero(owned[r])[0]) == [k for k in range(n) if k % world == r]


