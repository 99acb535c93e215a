"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every
entry point include/knor_b200.h declares (CPU only: no compute calls)."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "knor_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(knb_\w+)\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1606_08905_b200 import _native
    lib = _native.lib()
    names = declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.knb_version() == 1
    # every declared symbol has a Python binding signature (or is version/last_error)
    unbound = [n for n in names if n not in _native.SIGNATURES and n not in ("knb_version", "knb_last_error", "knb_f32_supported",
                                                                          "knb_mti_compact_ok")]
    assert not unbound, unbound


def test_library_is_sm100a_and_has_no_cpu_path():
    so = os.path.join(ROOT, "paper_1606_08905_b200", "libknorb200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out
    nm = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = re.findall(r"\bknb_\w+", nm)
    assert set(exported) == set(declared())


def test_error_path_without_gpu_is_loud():
    """Creating a context with no device raises (no silent CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1606_08905_b200 import _native
    with pytest.raises((RuntimeError, ValueError)):
        _native.Context(0, 10, 10, 0, 2, 2, False, 5, 0.0)


def test_f32_path_rule():
    """The f32 tensor-core path (config 5) applies to dense runs with 32 <= d <= 256,
    d % 4 == 0; everything else is upcast to f64 like the reference's check_matrix."""
    from paper_1606_08905_b200 import _native
    assert _native.f32_supported(256, 1000, False)
    assert _native.f32_supported(32, 8, False)
    assert not _native.f32_supported(256, 1000, True)
    assert not _native.f32_supported(16, 8, False)
    assert not _native.f32_supported(258, 8, False)
    assert not _native.f32_supported(260, 8, False)


def test_compacted_mti_kernel_dispatch_guard():
    """The compacted MTI kernel's filter uses 32-bit row indices: shards above
    2^31 - 2^26 rows must be routed to the block-dense pass."""
    from paper_1606_08905_b200 import _native
    assert _native.mti_compact_ok(856_000_000)
    assert _native.mti_compact_ok((1 << 31) - (1 << 26))
    assert not _native.mti_compact_ok((1 << 31) - (1 << 26) + 1)
    assert not _native.mti_compact_ok(3_000_000_000)
