"""CPU-side checks of the C-ABI library: it loads without a GPU and exports
every function include/specbatch_b200.h declares; host-only helpers agree
with the oracle."""

import re
from pathlib import Path

import numpy as np
import pytest

from oracle import spec_ref

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "specbatch_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2310_18813_b200 import _native

    lib = _native.load()
    declared = _declared()
    assert len(declared) >= 14
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared) <= set(_native.EXPORTED) | {"sb_init"}
    import re
    want = int(re.search(r"#define SB_ABI_VERSION (\d+)", (ROOT / 'include' / 'specbatch_b200.h').read_text()).group(1))
    assert lib.sb_version() == want
    assert b"sm_100a" in lib.sb_build_info()


def test_host_counter_rng_matches_oracle():
    from paper_2310_18813_b200 import _native

    lib = _native.load()
    for seed, stream, ctr in [(0, 0, 0), (9, 5, 130), (2**40 + 7, 123456, 64 * 99 + 3)]:
        assert np.float32(lib.sb_uniform_host(seed, stream, ctr)) == spec_ref.u01(seed, stream, ctr)


def test_missing_library_fails_loudly(tmp_path):
    from paper_2310_18813_b200 import _native
    from paper_2310_18813_b200.errors import NativeError

    saved = _native._lib
    try:
        _native._lib = None
        with pytest.raises(NativeError):
            _native.load(tmp_path / "nope.so")
    finally:
        _native._lib = saved
