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
    return set(re.findall(r"\b(pfw_[a-z_]+)\s*\(", text))


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
