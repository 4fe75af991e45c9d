"""The C-ABI library (no GPU needed): it loads, exports every function that
include/apbf_gpu.h declares, and the ctypes mirror has the exact C layout."""
import ctypes as C
import os
import subprocess
import tempfile

import pytest

from paper_1608_04721_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_reports_abi():
    lib = capi.load()
    assert lib.apbf_gpu_abi_version() == 1


def test_every_header_symbol_is_exported_and_bound():
    lib = capi.load()
    declared = capi.header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/apbf_gpu.h but not exported"
        assert name in capi.SIGNATURES, f"{name} has no ctypes signature"
    nm = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True, text=True)
    exported = {l.split()[-1] for l in nm.stdout.splitlines() if " T " in l}
    assert set(declared) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", capi.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_when_library_missing(monkeypatch):
    monkeypatch.setattr(capi, "_LIB", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        capi.load("/nonexistent/libapbf_gpu.so")


STRUCTS = ["apbf_error", "apbf_solver_config", "apbf_sdf_primitive", "apbf_camera",
           "apbf_lod_config", "apbf_frame_stats"]


def test_ctypes_layout_matches_header():
    src = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{ROOT}/include/apbf_gpu.h"',
           "int main(void) {"]
    for s in STRUCTS:
        src.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f, _ in getattr(capi, s)._fields_:
            cf = "pass" if f == "pass_" else f
            src.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {cf}));')
    src.append("return 0; }")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "layout.c")
        exe = os.path.join(d, "layout")
        open(c, "w").write("\n".join(src))
        subprocess.run(["gcc", "-o", exe, c], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.splitlines())
    for s in STRUCTS:
        cls = getattr(capi, s)
        assert int(got[s]) == C.sizeof(cls), s
        for f, _ in cls._fields_:
            assert int(got[f"{s}.{f}"]) == getattr(cls, f).offset, f"{s}.{f}"


def test_device_count_without_gpu_is_zero_or_more():
    assert capi.load().apbf_gpu_device_count() >= 0
