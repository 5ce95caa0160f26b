"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a,
loads, and exports every entry point include/quantspec_b200.h declares.
No kernel is launched (there is no GPU here)."""

import ctypes
import os
import re
import subprocess

import pytest

from .conftest import ROOT

HEADER = os.path.join(ROOT, "include", "quantspec_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qs_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2502_10424_b200 import _build

    return _build.build()


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("qs_encode_plane_hierarchical", "qs_kv_flush", "qs_attn_decode", "qs_linear", "qs_greedy_accept"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header(lib_path):
    from paper_2502_10424_b200 import _lib

    assert set(declared_symbols()) == set(_lib.EXPORTED)
    _lib.load()


def test_cubin_is_sm100a_and_uses_tensor_cores(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    # the decode contractions run as mma.sync (HMMA): at their N <= 48 columns a tcgen05 UMMA issues
    # no faster (profiles/r02/umma_rate.txt: ~45 cycles per m128 k16 UMMA, <= 2160 MAC/cycle/SM vs
    # 2048 for HMMA.16816); tensor memory holds the wide-query verify's parked accumulators
    assert "HMMA" in sass
    assert "LDTM" in sass and "STTM" in sass  # tcgen05.ld / tcgen05.st (TMEM accumulator parking)
    assert "UTCATOMSWS" in sass  # tcgen05.alloc / dealloc
    assert "UBLKCP" in sass  # TMA bulk copies staging the packed KV planes and weights


def test_status_codes_map_to_reference_errors(lib_path):
    from paper_2502_10424_b200 import _lib, errors

    with pytest.raises(errors.ConfigError):
        _lib.check(2, "x")
    with pytest.raises(errors.BufferOverflowError):
        _lib.check(5, "x")
    assert issubclass(errors.BufferOverflowError, errors.CacheIntegrityError)
