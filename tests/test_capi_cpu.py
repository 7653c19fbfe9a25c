"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/bitdelta/capi.h declares; status codes mirror deltakit::errc;
calls that fail validation return the right category without touching a GPU."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "bitdelta", "capi.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bd_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_api():
    syms = declared_symbols()
    for s in ["bd_compress", "bd_compress_batched", "bd_packed_signed_accumulate", "bd_packed_matvec",
              "bd_multitenant_linear", "bd_pool_create", "bd_pool_decode_step", "bd_pool_decode_layers"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2402_10193_b200 import capi

    if not os.path.exists(capi.LIB_PATH):
        from paper_2402_10193_b200 import build

        build.build()
    lib = C.CDLL(capi.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(capi.SYMBOLS) <= set(declared_symbols())
    assert lib.bd_abi_version() == 1


def test_status_codes_mirror_errc():
    """BD_ERR_* == 1 + deltakit::errc enumerator (P:include/deltakit/error.hpp:10-25)."""
    errc = ["io", "malformed_header", "json_parse", "bad_offsets", "unsupported_dtype", "shape_mismatch",
            "name_mismatch", "length_mismatch", "bad_argument", "bad_token", "non_finite",
            "no_convergence", "duplicate_id", "unknown_id"]
    text = open(HEADER).read()
    for i, name in enumerate(errc):
        m = re.search(r"BD_ERR_%s\s*=\s*(\d+)" % name.upper(), text)
        assert m and int(m.group(1)) == i + 1, name
    from paper_2402_10193_b200.capi import ERRC

    assert [ERRC[i + 1] for i in range(14)] == errc


def test_validation_errors_without_gpu():
    """Argument validation happens before any device work."""
    from paper_2402_10193_b200 import capi

    lib = capi.lib()
    assert lib.bd_packed_size(3, 3) == 2 and lib.bd_packed_size(0, 5) == 0
    rc = lib.bd_compress_batched(None, 1, 0, None)
    assert rc == 9  # bad_argument
    assert b"null" in lib.bd_last_error()
    rc = lib.bd_compress(None, None, 7, 2, 2, None, None, None)
    assert rc == 5  # unsupported_dtype
    rc = lib.bd_device_check(0)
    assert rc in (101, 102) or rc == 0  # no device here -> no_device


def test_tensor_shapes_match_reference_order():
    """serving.tensor_shapes == arch.cpp:51-69 ordering (checked against the reference when built)."""
    import json

    import oracle
    from paper_2402_10193_b200.serving import tensor_shapes

    arch = {"vocab": 48, "dim": 32, "n_layers": 2, "n_heads": 4, "intermediate": 40, "max_seq": 32}
    mine = tensor_shapes(arch)
    assert mine[0] == ("embed", 48, 32) and mine[-1] == ("lm_head", 48, 32) and len(mine) == 21
    if oracle.have_ref():
        cfg = json.dumps(dict(arch, rope_theta=10000.0))
        assert [tuple(t) for t in oracle.ref().tensor_specs(cfg)] == mine
