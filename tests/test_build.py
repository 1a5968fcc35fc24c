"""CPU checks of the native artefacts: the C ABI library exports every symbol
include/mpcd.h declares, its signatures table matches the header, the
numerics contract (no FMA contraction) holds in the PTX, and the host-side
helpers of the library agree with the oracle.  No GPU needed."""

import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from paper_2212_11878_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpcd.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mpcd_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    out = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mpcd_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_ctypes_table_covers_header(lib):
    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_version_and_error_strings(lib):
    assert b"sm_100a" in lib.mpcd_version()
    assert lib.mpcd_last_error() is not None


def test_no_fma_contraction_in_parity_kernels():
    """-fmad=false: numpy never fuses a*b+c.  PTX-level fma.rn.f64 may only
    come from libdevice transcendentals of the (non-bit-exact) device init."""
    src = [os.path.join(_build.CSRC, f) for f in os.listdir(_build.CSRC) if f.endswith(".cu")]
    for path in src:
        ptx = subprocess.run(
            [_build.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false",
             "-std=c++17", "-I", _build.INCLUDE, "-I", _build.CSRC, "-ptx", "-o", "-", path],
            capture_output=True, text=True, check=True).stdout
        entry = None
        for line in ptx.splitlines():
            m = re.search(r"\.entry\s+(\S+)\(", line)
            if m:
                entry = m.group(1)
            if "fma.rn.f64" in line:
                assert entry is not None and ("k_init_sum" in entry or "k_init_place" in entry), \
                    (path, entry)


def test_host_rng_helpers_match_oracle(lib):
    rs = np.random.default_rng(0)
    for _ in range(50):
        k = [int(x) for x in rs.integers(0, 2 ** 63, size=4)]
        assert lib.mpcd_key_state(*k) == oracle.key_state(*k)
        st = lib.mpcd_key_state(*k)
        assert lib.mpcd_uniform_at(st, k[0]) == oracle.uniform_at(st, k[0])
    import ctypes as C
    out = (C.c_double * 3)()
    for kind, kid in _lib.PRNGS.items():
        for step in range(10):
            lib.mpcd_grid_shift(kid, 42, step, 1.0, out)
            assert np.array_equal(np.array(out[:]), oracle.grid_shift(step, 42, 1.0, kind))


def test_sass_has_tma_and_mbarrier():
    """The step kernel streams tiles with cp.async.bulk (UBLKCP) on mbarriers."""
    _build.build()
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UBLKCP" in sass
    assert "SYNCS" in sass
    # one 256-bit store per 32-byte particle record (sm_100 STG.256)
    assert re.search(r"STG\.E\.[A-Z0-9.]*256", sass)
    # the fused migration's system-scope fence
    assert "MEMBAR" in sass
