"""The drop-in boundary: the C-ABI library exists, loads, and exports every symbol that
include/sgc_b200.h declares (no compute calls: this runs on the CPU box)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sgc_b200.h")
LIB = os.path.join(ROOT, "paper_2505_10951_b200", "libsgc_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sgc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("sgc_encode_subgraphs", "sgc_agglomerate", "sgc_build_representatives",
              "sgc_prefill", "sgc_extend", "sgc_run_subgcache", "sgc_last_error"):
        assert s in syms


def test_library_loads_and_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.fail("libsgc_b200.so not built: run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    from paper_2505_10951_b200 import _lib

    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_sass_has_tcgen05_and_tma():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out or "UTCQMMA" in out or "UTCMMA" in out  # tcgen05.mma
    assert "UTMALDG" in out                                           # TMA loads
    assert "LDTM" in out                                              # tcgen05.ld


def test_errors_map_to_reference_taxonomy():
    from paper_2505_10951_b200 import _lib

    assert issubclass(_lib.DomainError, ValueError)
    for code, exc in ((1, _lib.DomainError), (2, _lib.CapacityError), (3, _lib.IntegrityError),
                      (4, _lib.ParseError), (5, _lib.LogicError), (6, _lib.CudaError)):
        assert _lib._EXC[code] is exc


def test_no_device_without_gpu_fails_loudly():
    """On a machine without an sm_100 device the product path raises; it never falls back."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2505_10951_b200 import host

    with pytest.raises(host.CudaError):
        host.Context(0)
