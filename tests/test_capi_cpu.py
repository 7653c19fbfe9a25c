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


def _validate(path):
    from paper_2402_10193_b200 import capi

    n, k, mp = C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = capi.lib().bd_bdelta_validate(str(path).encode(), C.byref(n), C.byref(k), C.byref(mp))
    return rc, n.value, k.value, mp.value


def test_bdelta_reader_accepts_reference_files():
    """Files written by the reference's write_delta_file (tests/golden) parse on the host:
    the toy universe (1 plane) and the 2/3-plane universe."""
    from conftest import GOLDEN

    rc, n, k, mp = _validate(os.path.join(GOLDEN, "toy_t0.bdelta"))
    assert rc == 0 and n == 21 and k == 14 and mp == 1
    rc, n, k, mp = _validate(os.path.join(GOLDEN, "mp_t1.bdelta"))
    assert rc == 0 and k == 7 and mp == 3


def _rewrite_header(src, dst, transform):
    import struct

    b = open(src, "rb").read()
    hlen = struct.unpack("<I", b[8:12])[0]
    header = transform(b[12:12 + hlen])
    open(dst, "wb").write(b[:8] + struct.pack("<I", len(header)) + header + b[12 + hlen:])


def test_bdelta_reader_rejects_like_read_delta_file(tmp_path):
    """read_delta_file (nlohmann) semantics: trailing bytes after the JSON array, fractional
    sizes and bad escapes are json_parse errors; \\uXXXX escapes decode."""
    import json

    from conftest import GOLDEN

    src = os.path.join(GOLDEN, "toy_t0.bdelta")
    p = tmp_path / "x.bdelta"
    _rewrite_header(src, p, lambda h: h + b" ]")
    assert _validate(p)[0] == 3  # json_parse
    _rewrite_header(src, p, lambda h: h.replace(b'"rows":1,', b'"rows":1.5,', 1))
    assert _validate(p)[0] == 3
    _rewrite_header(src, p, lambda h: h.replace(b'"embed"', b'"emb\\q"', 1))
    assert _validate(p)[0] == 3

    def rename(h):  # "embed" spelled with \u escapes: same name, parses
        j = json.loads(h)
        s = json.dumps(j).replace('"embed"', '"\\u0065mbed"', 1)
        return s.encode()

    _rewrite_header(src, p, rename)
    assert _validate(p)[0] == 0
    open(p, "wb").write(b"BDLT\x02\x00\x00\x00\x00\x00\x00\x00")
    assert _validate(p)[0] == 2  # malformed_header (version)


def test_doctest_shim_runs_reference_suites_on_the_reference():
    """Control for tests/test_gpu_reference_suites.py: the same unchanged reference suites
    through the doctest shim against the unmodified reference library (no GPU) all pass."""
    import subprocess

    exe = os.path.join(ROOT, "integration", "_build", "deltakit_tests_ref")
    if not os.path.exists(exe):
        pytest.skip("integration/_build not built (reference sources absent)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "[doctest] test cases: 39 passed, 0 failed, 0 skipped" in r.stdout, r.stdout[-3000:]
