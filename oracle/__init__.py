"""TEST INFRASTRUCTURE — the parity checkers. NOT PART OF THE PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the timed CPU baseline — never as the thing measured or
shipped. The product (``paper_2402_10193_b200``) never imports it.

Two checkers, both loaded with ctypes:

* ``ref()``  — the UNMODIFIED reference library (deltakit), compiled from
  /root/reference/proj/src by ``oracle/Makefile`` into ``oracle/_ref/`` and
  wrapped by ``oracle/ref_shim.cpp``. This is the ground truth.
* ``port()`` — ``oracle/bdoracle.c``, a plain-C restatement of the same path
  with file:line citations; pinned against ``ref()`` and the golden vectors by
  ``tests/test_oracle.py``.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libdeltakit_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libbdoracle.so")

u64 = C.c_uint64
f32p = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)


def _p(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def build() -> None:
    """Build both checkers (the reference only where /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def have_ref() -> bool:
    return os.path.exists(REF_SO)


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"deltakit error {code}: {msg}")
        self.code = code


@lru_cache(maxsize=None)
def _ref_lib():
    if not os.path.exists(REF_SO):
        raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
    lib = C.CDLL(REF_SO)
    lib.dkref_last_error.restype = C.c_char_p
    lib.dkref_packed_size.restype = u64
    lib.dkref_packed_size.argtypes = [u64, u64]
    lib.dkref_rmsnorm_row.restype = C.c_double
    lib.dkref_silu.restype = C.c_float
    lib.dkref_silu.argtypes = [C.c_float]
    lib.dkref_sign_of.argtypes = [C.c_float]
    lib.dkref_pool_backbone_passes.restype = u64
    lib.dkref_pool_backbone_passes.argtypes = [C.c_void_p]
    lib.dkref_pool_destroy.argtypes = [C.c_void_p]
    return lib


@lru_cache(maxsize=None)
def _port_lib():
    if not os.path.exists(PORT_SO):
        raise FileNotFoundError(f"{PORT_SO} not built (make -C oracle port)")
    lib = C.CDLL(PORT_SO)
    lib.bdo_packed_size.restype = u64
    lib.bdo_packed_size.argtypes = [u64, u64]
    lib.bdo_rmsnorm_row.restype = C.c_double
    lib.bdo_silu.restype = C.c_float
    lib.bdo_silu.argtypes = [C.c_float]
    lib.bdo_sign_of.argtypes = [C.c_float]
    lib.bdo_tensor_count.restype = u64
    return lib


def packed_size(rows: int, cols: int) -> int:
    return (rows * cols + 7) // 8


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


class _Common:
    """Shared numpy-facing API; subclasses bind the symbols."""

    def compress_delta(self, delta: np.ndarray):
        d = _f32(delta)
        rows, cols = d.shape
        bits = np.zeros(packed_size(rows, cols), np.uint8)
        scale = C.c_float()
        self._compress_delta(d, rows, cols, bits, scale)
        return bits, np.float32(scale.value)

    def compress_tensor(self, base: np.ndarray, fine: np.ndarray):
        b, f = _f32(base), _f32(fine)
        rows, cols = b.shape
        bits = np.zeros(packed_size(rows, cols), np.uint8)
        scale = C.c_float()
        self._compress_tensor(b, f, rows, cols, bits, scale)
        return bits, np.float32(scale.value)

    def compress_stack(self, base, fine, planes: int):
        b, f = _f32(base), _f32(fine)
        rows, cols = b.shape
        bits = np.zeros(planes * packed_size(rows, cols), np.uint8)
        scales = np.zeros(planes, np.float32)
        self._compress_stack(b, f, rows, cols, planes, bits, scales)
        return bits.reshape(planes, -1), scales

    def decompress(self, bits, rows: int, cols: int, scale: float) -> np.ndarray:
        out = np.zeros((rows, cols), np.float32)
        self._decompress(np.ascontiguousarray(bits, np.uint8), rows, cols, scale, out)
        return out

    def packed_signed_accumulate(self, bits, rows: int, cols: int, x, out=None) -> np.ndarray:
        x = _f32(x)
        out = np.zeros(rows, np.float32) if out is None else _f32(out).copy()
        self._psa(np.ascontiguousarray(bits, np.uint8), rows, cols, x, out)
        return out

    def packed_signed_accumulate_t(self, bits, rows: int, cols: int, y, out=None) -> np.ndarray:
        y = _f32(y)
        out = np.zeros(cols, np.float32) if out is None else _f32(out).copy()
        self._psat(np.ascontiguousarray(bits, np.uint8), rows, cols, y, out)
        return out

    def packed_matvec(self, bits, rows: int, cols: int, scale: float, x) -> np.ndarray:
        y = np.zeros(rows, np.float32)
        self._pmv(np.ascontiguousarray(bits, np.uint8), rows, cols, scale, _f32(x), y)
        return y

    def rtn_quantize(self, w):
        w = _f32(w)
        rows, cols = w.shape
        q = np.zeros((rows, cols), np.int8)
        sc = np.zeros(rows, np.float32)
        self._rtn(w, rows, cols, q, sc)
        return q, sc

    def int8_matmul_nt(self, a, q, scales) -> np.ndarray:
        a = _f32(a)
        q = np.ascontiguousarray(q, np.int8)
        out = np.zeros((a.shape[0], q.shape[0]), np.float32)
        self._i8mm(a, a.shape[0], q, _f32(scales), q.shape[0], q.shape[1], out)
        return out

    def matmul_nt(self, a, b) -> np.ndarray:
        a, b = _f32(a), _f32(b)
        out = np.zeros((a.shape[0], b.shape[0]), np.float32)
        self._mmnt(a, a.shape[0], a.shape[1], b, b.shape[0], out)
        return out


class Ref(_Common):
    """ctypes facade over oracle/_ref/libdeltakit_ref.so (the reference itself)."""

    def __init__(self):
        self.lib = _ref_lib()

    def _chk(self, rc: int):
        if rc != 0:
            raise RefError(rc, self.lib.dkref_last_error().decode())

    def sign_of(self, x: float) -> int:
        return self.lib.dkref_sign_of(x)

    def _compress_delta(self, d, rows, cols, bits, scale):
        self._chk(self.lib.dkref_compress_delta(_p(d, C.c_float), u64(rows), u64(cols), _p(bits, C.c_uint8), C.byref(scale)))

    def _compress_tensor(self, b, f, rows, cols, bits, scale):
        self._chk(self.lib.dkref_compress_tensor(_p(b, C.c_float), _p(f, C.c_float), u64(rows), u64(cols), _p(bits, C.c_uint8), C.byref(scale)))

    def _compress_stack(self, b, f, rows, cols, planes, bits, scales):
        self._chk(self.lib.dkref_compress_stack(_p(b, C.c_float), _p(f, C.c_float), u64(rows), u64(cols), u64(planes), _p(bits, C.c_uint8), _p(scales, C.c_float)))

    def _decompress(self, bits, rows, cols, scale, out):
        self._chk(self.lib.dkref_decompress(_p(bits, C.c_uint8), u64(rows), u64(cols), C.c_float(scale), _p(out, C.c_float)))

    def _psa(self, bits, rows, cols, x, out):
        self._chk(self.lib.dkref_packed_signed_accumulate(_p(bits, C.c_uint8), u64(rows), u64(cols), _p(x, C.c_float), _p(out, C.c_float)))

    def _rtn(self, w, rows, cols, q, sc):
        self._chk(self.lib.dkref_rtn_quantize(_p(w, C.c_float), u64(rows), u64(cols), _p(q, C.c_int8), _p(sc, C.c_float)))

    def _i8mm(self, a, s, q, sc, rows, cols, out):
        self._chk(self.lib.dkref_int8_matmul_nt(_p(a, C.c_float), u64(s), _p(q, C.c_int8), _p(sc, C.c_float), u64(rows), u64(cols), _p(out, C.c_float)))

    def _psat(self, bits, rows, cols, y, out):
        self._chk(self.lib.dkref_packed_signed_accumulate_t(_p(bits, C.c_uint8), u64(rows), u64(cols), _p(y, C.c_float), _p(out, C.c_float)))

    def _pmv(self, bits, rows, cols, scale, x, y):
        self._chk(self.lib.dkref_packed_matvec(_p(bits, C.c_uint8), u64(rows), u64(cols), C.c_float(scale), _p(x, C.c_float), _p(y, C.c_float)))

    def _mmnt(self, a, s, k, b, t, out):
        self._chk(self.lib.dkref_matmul_nt(_p(a, C.c_float), u64(s), u64(k), _p(b, C.c_float), u64(t), _p(out, C.c_float)))

    def rmsnorm_row(self, x, w):
        x, w = _f32(x), _f32(w)
        out = np.zeros_like(x)
        self.lib.dkref_rmsnorm_row(_p(x, C.c_float), _p(w, C.c_float), u64(x.size), _p(out, C.c_float))
        return out

    def rope_row(self, head, pos: int, theta: float):
        h = _f32(head).copy()
        self.lib.dkref_rope_row(_p(h, C.c_float), u64(h.size), u64(pos), C.c_float(theta))
        return h

    def softmax_row(self, row):
        r = _f32(row).copy()
        self.lib.dkref_softmax_row(_p(r, C.c_float), u64(r.size))
        return r

    # ---- model-level (toy configs) ----
    def tensor_specs(self, cfg_json: str):
        n = u64()
        self._chk(self.lib.dkref_tensor_count(cfg_json.encode(), C.byref(n)))
        out = []
        buf = C.create_string_buffer(256)
        for i in range(n.value):
            r, c = u64(), u64()
            self._chk(self.lib.dkref_tensor_spec(cfg_json.encode(), u64(i), buf, u64(256), C.byref(r), C.byref(c)))
            out.append((buf.value.decode(), r.value, c.value))
        return out

    def synth_base(self, cfg_json: str, seed: int, weight_scale: float = 0.08) -> np.ndarray:
        total = sum(r * c for _, r, c in self.tensor_specs(cfg_json))
        out = np.zeros(total, np.float32)
        self._chk(self.lib.dkref_synth_base(cfg_json.encode(), u64(seed), C.c_float(weight_scale), _p(out, C.c_float)))
        return out

    def synth_fine(self, cfg_json: str, base: np.ndarray, magnitude: float, seed: int, signed=False) -> np.ndarray:
        base = _f32(base)
        out = np.zeros_like(base)
        self._chk(self.lib.dkref_synth_fine(cfg_json.encode(), _p(base, C.c_float), C.c_int(1 if signed else 0), C.c_float(magnitude), u64(seed), _p(out, C.c_float)))
        return out

    def write_delta_file(self, cfg_json: str, base, fine, planes: int, path: str):
        base, fine = _f32(base), _f32(fine)
        self._chk(self.lib.dkref_write_delta_file(cfg_json.encode(), _p(base, C.c_float), _p(fine, C.c_float), u64(planes), path.encode()))

    def pool(self, cfg_json: str, base) -> "RefPool":
        return RefPool(self, cfg_json, _f32(base))


class RefPool:
    """The reference ServingPool (serve.hpp:59-125) behind ctypes."""

    def __init__(self, ref: Ref, cfg_json: str, base: np.ndarray):
        import json

        self.ref = ref
        self.vocab = json.loads(cfg_json)["vocab"]
        self.h = C.c_void_p()
        ref._chk(ref.lib.dkref_pool_create(cfg_json.encode(), _p(base, C.c_float), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.dkref_pool_destroy(self.h)
            self.h = None

    def register_delta(self, id_: str, path: str, resident: bool = True):
        self.ref._chk(self.ref.lib.dkref_pool_register(self.h, id_.encode(), path.encode(), C.c_int(int(resident))))

    def open_request(self, id_: str) -> int:
        r = u64()
        self.ref._chk(self.ref.lib.dkref_pool_open(self.h, id_.encode(), C.byref(r)))
        return r.value

    def decode_step(self, reqs, naive: bool = False) -> np.ndarray:
        """reqs: list of (request_id, token, position)."""
        n = len(reqs)
        ids = np.array([r[0] for r in reqs], np.uint64)
        toks = np.array([r[1] for r in reqs], np.int32)
        pos = np.array([r[2] for r in reqs], np.uint64)
        out = np.zeros((n, self.vocab), np.float32)
        self.ref._chk(self.ref.lib.dkref_pool_decode(self.h, u64(n), _p(ids, C.c_uint64), _p(toks, C.c_int32), _p(pos, C.c_uint64), C.c_int(int(naive)), _p(out, C.c_float)))
        return out

    @property
    def backbone_passes(self) -> int:
        return self.ref.lib.dkref_pool_backbone_passes(self.h)


class Port(_Common):
    """ctypes facade over oracle/_build/libbdoracle.so (the C restatement)."""

    def __init__(self):
        self.lib = _port_lib()

    def sign_of(self, x: float) -> int:
        return self.lib.bdo_sign_of(x)

    def _compress_delta(self, d, rows, cols, bits, scale):
        self.lib.bdo_compress_delta(_p(d, C.c_float), u64(rows * cols), _p(bits, C.c_uint8), C.byref(scale))

    def _compress_tensor(self, b, f, rows, cols, bits, scale):
        self.lib.bdo_compress_tensor(_p(b, C.c_float), _p(f, C.c_float), u64(rows * cols), _p(bits, C.c_uint8), C.byref(scale))

    def _compress_stack(self, b, f, rows, cols, planes, bits, scales):
        self.lib.bdo_compress_stack(_p(b, C.c_float), _p(f, C.c_float), u64(rows * cols), u64(planes), _p(bits, C.c_uint8), _p(scales, C.c_float))

    def _decompress(self, bits, rows, cols, scale, out):
        self.lib.bdo_decompress(_p(bits, C.c_uint8), u64(rows * cols), C.c_float(scale), _p(out, C.c_float))

    def _psa(self, bits, rows, cols, x, out):
        self.lib.bdo_packed_signed_accumulate(_p(bits, C.c_uint8), u64(rows), u64(cols), _p(x, C.c_float), _p(out, C.c_float))

    def _rtn(self, w, rows, cols, q, sc):
        self.lib.bdo_rtn_quantize(_p(w, C.c_float), u64(rows), u64(cols), _p(q, C.c_int8), _p(sc, C.c_float))

    def _i8mm(self, a, s, q, sc, rows, cols, out):
        self.lib.bdo_int8_matmul_nt(_p(a, C.c_float), u64(s), _p(q, C.c_int8), _p(sc, C.c_float), u64(rows), u64(cols), _p(out, C.c_float))

    def _psat(self, bits, rows, cols, y, out):
        self.lib.bdo_packed_signed_accumulate_t(_p(bits, C.c_uint8), u64(rows), u64(cols), _p(y, C.c_float), _p(out, C.c_float))

    def _pmv(self, bits, rows, cols, scale, x, y):
        self.lib.bdo_packed_matvec(_p(bits, C.c_uint8), u64(rows), u64(cols), C.c_float(scale), _p(x, C.c_float), _p(y, C.c_float))

    def _mmnt(self, a, s, k, b, t, out):
        self.lib.bdo_matmul_nt(_p(a, C.c_float), u64(s), u64(k), _p(b, C.c_float), u64(t), _p(out, C.c_float))

    def rmsnorm_row(self, x, w):
        x, w = _f32(x), _f32(w)
        out = np.zeros_like(x)
        self.lib.bdo_rmsnorm_row(_p(x, C.c_float), _p(w, C.c_float), u64(x.size), _p(out, C.c_float))
        return out

    def rope_row(self, head, pos: int, theta: float):
        h = _f32(head).copy()
        self.lib.bdo_rope_row(_p(h, C.c_float), u64(h.size), u64(pos), C.c_float(theta))
        return h

    def softmax_row(self, row):
        r = _f32(row).copy()
        self.lib.bdo_softmax_row(_p(r, C.c_float), u64(r.size))
        return r

    def decode(self, arch: dict, base: np.ndarray, tenant_entries, req_tenant, tokens, pos,
               kcache, vcache, layers_only=False, x_in=None):
        """decode_shared restatement. tenant_entries[t] = list (tensor order) of
        dicts {kind: 'packed'|'raw', bits: uint8[planes, nb], scales: f32[planes], raw: f32}.
        kcache/vcache: per request f32 [n_layers, max_seq, kv_dim] (mutated)."""
        A = _Arch(**arch)
        keep = []
        tables = []
        for ents in tenant_entries:
            arr = (_Entry * len(ents))()
            for i, e in enumerate(ents):
                if e["kind"] == "packed":
                    b = np.ascontiguousarray(e["bits"], np.uint8)
                    s = _f32(e["scales"])
                    keep += [b, s]
                    arr[i] = _Entry(1, len(s), _p(b, C.c_uint8), _p(s, C.c_float), None)
                else:
                    r = _f32(e["raw"])
                    keep.append(r)
                    arr[i] = _Entry(0, 0, None, None, _p(r, C.c_float))
            tables.append(arr)
        B = len(req_tenant)
        ents_pp = (C.POINTER(_Entry) * B)(*[C.cast(tables[t], C.POINTER(_Entry)) for t in req_tenant])
        base = _f32(base)
        kp = (f32p * B)(*[_p(k, C.c_float) for k in kcache])
        vp = (f32p * B)(*[_p(v, C.c_float) for v in vcache])
        posa = np.ascontiguousarray(pos, np.uint64)
        if layers_only:
            xin = _f32(x_in)
            out = np.zeros((B, A.dim), np.float32)
            rc = self.lib.bdo_decode_layers(C.byref(A), _p(base, C.c_float), ents_pp, u64(B), _p(posa, C.c_uint64), kp, vp, _p(xin, C.c_float), _p(out, C.c_float))
        else:
            toks = np.ascontiguousarray(tokens, np.int32)
            out = np.zeros((B, A.vocab), np.float32)
            rc = self.lib.bdo_decode_shared(C.byref(A), _p(base, C.c_float), ents_pp, u64(B), _p(toks, C.c_int32), _p(posa, C.c_uint64), kp, vp, _p(out, C.c_float))
        if rc != 0:
            raise ValueError(f"bdo_decode rc={rc}")
        return out


class _Arch(C.Structure):
    _fields_ = [("vocab", u64), ("dim", u64), ("kv_dim", u64), ("n_layers", u64), ("n_heads", u64),
                ("intermediate", u64), ("max_seq", u64), ("rope_theta", C.c_float)]


class _Entry(C.Structure):
    _fields_ = [("kind", C.c_int), ("planes", u64), ("bits", u8p), ("scales", f32p), ("raw", f32p)]


@lru_cache(maxsize=None)
def ref() -> Ref:
    return Ref()


@lru_cache(maxsize=None)
def port() -> Port:
    return Port()
