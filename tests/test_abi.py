"""The C-ABI library: it loads without a GPU, exports every symbol that
include/pfw.h declares, and the product path fails loudly without a device."""
from __future__ import annotations

import os
import re

import pytest

from conftest import ROOT, gpu_available
from paper_1312_4188_b200 import _native


def header_symbols() -> set[str]:
    text = open(os.path.join(ROOT, "include", "pfw.h")).read()
    return set(re.findall(r"\b(pfw_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_header_symbol():
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"libpfw.so does not export {s}"
    assert set(_native.EXPORTS) == syms


def test_version_and_tuning_validation():
    assert "sm_100a" in _native.version()
    with pytest.raises(ValueError):
        _native.set_tuning("ks", 3)
    with pytest.raises(ValueError):
        _native.set_tuning("bogus", 1)


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_no_silent_cpu_fallback():
    import paper_1312_4188_b200 as pfw
    assert _native.device_count() == 0
    with pytest.raises(_native.NativeUnavailable):
        pfw.CompiledRuleset(pfw.Ruleset())
    rs = pfw.generate_ruleset(pfw.RulesetGenParams(4, 1))
    pk = [pfw.Packet(0, pfw.Protocol.TCP, 1, 2, 3, 4)]
    with pytest.raises(_native.NativeUnavailable):
        pfw.classify_batch_sequential(rs, pk)


def test_non_prefix_masks_are_rejected():
    """Masks must be CIDR prefix masks (model.py:108-114); both encodings of
    the CIDR test are exact only for those, so anything else is refused
    before any device work (this runs without a GPU)."""
    import ctypes
    import numpy as np
    lib = _native.load()
    cols = [np.array([6], np.uint8), np.array([0x0A000000], np.uint32), np.array([0xFF00FF00], np.uint32),
            np.array([0], np.uint16), np.array([65535], np.uint16), np.array([0], np.uint32),
            np.array([0], np.uint32), np.array([0], np.uint16), np.array([65535], np.uint16),
            np.array([1], np.uint8)]
    h = ctypes.c_void_p()
    rc = lib.pfw_ruleset_create(0, 1, *[c.ctypes.data for c in cols], ctypes.byref(h))
    assert rc == _native.PFW_ERR_INVALID
    assert "not a prefix mask" in _native.last_error()
