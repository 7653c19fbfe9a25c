"""B200-native BitDelta hot path (compress + multi-tenant decode), behind the
reference deltakit API.

Host-side Python mirror of the reference operators over the C-ABI in
include/bitdelta/capi.h. PyTorch is used only for device memory and streams;
all compute runs in libbitdelta_b200.so (sm_100a). Names, argument meaning and
error categories follow deltakit (P:include/deltakit/delta.hpp, serve.hpp).
"""
from __future__ import annotations

import ctypes as C

from .capi import (BD_BF16, BD_F32, Arch, BitDeltaError, CompressJob, DeltaEntry, PoolStats,
                   Request, check, lib)

__all__ = [
    "BitDeltaError", "packed_size", "compress_tensor", "compress_delta", "compress_batched",
    "compress_stack", "packed_signed_accumulate", "packed_matvec", "multitenant_linear",
    "ServingPool", "device_check", "launch_count",
]


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _dtype(t) -> int:
    import torch

    if t.dtype == torch.float32:
        return BD_F32
    if t.dtype == torch.bfloat16:
        return BD_BF16
    raise BitDeltaError(5, f"unsupported dtype {t.dtype}")


def device_check(device: int = 0) -> None:
    check(lib().bd_device_check(device))


def launch_count() -> int:
    return int(lib().bd_launch_count())


def packed_size(rows: int, cols: int) -> int:
    """PackedSignMatrix::packed_size (delta.hpp:28-30)."""
    return (rows * cols + 7) // 8


def _req_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise BitDeltaError(9, "tensors must live on the CUDA device (no CPU fallback)")


def compress_tensor(base, fine, stream=None):
    """compress_tensor (delta.hpp:48): bits (uint8[ceil(n/8)]) and alpha (f32[1]) on device."""
    import torch

    _req_cuda(base, fine)
    if base is not None and base.shape != fine.shape:
        raise BitDeltaError(6, "compress_tensor: shape mismatch")
    rows, cols = fine.shape
    bits = torch.empty(packed_size(rows, cols), dtype=torch.uint8, device=fine.device)
    alpha = torch.empty(1, dtype=torch.float32, device=fine.device)
    b = base.contiguous() if base is not None else None
    f = fine.contiguous()
    if b is not None and b.dtype != f.dtype:
        raise BitDeltaError(5, "compress_tensor: base/fine dtypes differ")
    check(lib().bd_compress(_ptr(b), _ptr(f), _dtype(f), rows, cols, _ptr(bits), _ptr(alpha), _stream(stream)))
    return bits, alpha


def compress_delta(delta, stream=None):
    """compress_delta (delta.hpp:47)."""
    return compress_tensor(None, delta, stream)


def compress_batched(pairs, stream=None, outs=None):
    """Many (base, fine) pairs of one dtype in a single launch; returns [(bits, alpha)]
    (written into `outs` when given: [(uint8[packed_size], f32[1])] per pair)."""
    import torch

    jobs = (CompressJob * len(pairs))()
    given, outs, keep = outs, [], []
    dt = None
    for i, (b, f) in enumerate(pairs):
        _req_cuda(b, f)
        f = f.contiguous()
        b = b.contiguous() if b is not None else None
        dt = _dtype(f) if dt is None else dt
        if _dtype(f) != dt:
            raise BitDeltaError(5, "compress_batched: mixed dtypes")
        rows, cols = f.shape
        if given is not None:
            bits, alpha = given[i]
            if bits.numel() != packed_size(rows, cols) or not bits.is_cuda or not alpha.is_cuda:
                raise BitDeltaError(8, "compress_batched: output buffer of the wrong size")
        else:
            bits = torch.empty(packed_size(rows, cols), dtype=torch.uint8, device=f.device)
            alpha = torch.empty(1, dtype=torch.float32, device=f.device)
        jobs[i] = CompressJob(_ptr(b) or None, _ptr(f), rows, cols, _ptr(bits), _ptr(alpha))
        outs.append((bits, alpha))
        keep += [b, f]
    check(lib().bd_compress_batched(jobs, len(pairs), dt or BD_F32, _stream(stream)))
    return outs


def compress_stack(base, fine, planes: int, stream=None):
    """compress_stack (delta.hpp:62): (bits uint8[planes, nb], alphas f32[planes])."""
    import torch

    _req_cuda(base, fine)
    rows, cols = fine.shape
    nb = packed_size(rows, cols)
    bits = torch.empty((max(planes, 1), nb), dtype=torch.uint8, device=fine.device)
    alphas = torch.empty(max(planes, 1), dtype=torch.float32, device=fine.device)
    f = fine.contiguous()
    b = base.contiguous() if base is not None else None
    check(lib().bd_compress_stack(_ptr(b), _ptr(f), _dtype(f), rows, cols, planes, _ptr(bits),
                                  _ptr(alphas), _stream(stream)))
    return bits, alphas


def packed_signed_accumulate(bits, rows: int, cols: int, x, out, stream=None):
    """packed_signed_accumulate (delta.hpp:69-70): out += S x, for x of shape
    [cols] or [n_vec, cols] (f32, device). Accumulates in place into `out`."""
    _req_cuda(bits, x, out)
    n_vec = 1 if x.dim() == 1 else x.shape[0]
    if x.shape[-1] != cols or out.shape[-1] != rows or out.numel() != n_vec * rows:
        raise BitDeltaError(8, "packed_signed_accumulate: length mismatch")
    check(lib().bd_packed_signed_accumulate(_ptr(bits), rows, cols, _ptr(x.contiguous()), n_vec,
                                            _ptr(out), _stream(stream)))
    return out


def packed_matvec(bits, alpha: float, rows: int, cols: int, x, stream=None):
    """packed_matvec (delta.hpp:67): alpha * S x."""
    import torch

    _req_cuda(bits, x)
    if x.shape[-1] != cols:
        raise BitDeltaError(8, "packed_matvec: length mismatch")
    n_vec = 1 if x.dim() == 1 else x.shape[0]
    y = torch.empty((n_vec, rows) if x.dim() > 1 else (rows,), dtype=torch.float32, device=x.device)
    check(lib().bd_packed_matvec(_ptr(bits), float(alpha), rows, cols, _ptr(x.contiguous()), n_vec,
                                 _ptr(y), _stream(stream)))
    return y


def packed_signed_accumulate_t(bits, rows: int, cols: int, y, out, stream=None):
    """packed_signed_accumulate_t (delta.hpp:71-72, delta.cpp:105-131): out += S^T y, for y of
    shape [rows] or [n_vec, rows] (f32, device). Accumulates in place into `out`."""
    _req_cuda(bits, y, out)
    n_vec = 1 if y.dim() == 1 else y.shape[0]
    if y.shape[-1] != rows or out.shape[-1] != cols or out.numel() != n_vec * cols:
        raise BitDeltaError(8, "packed_signed_accumulate_t: length mismatch")
    check(lib().bd_packed_signed_accumulate_t(_ptr(bits), rows, cols, _ptr(y.contiguous()), n_vec, _ptr(out),
                                              _stream(stream)))
    return out


def delta_linear_backward(planes, scales, rows: int, cols: int, dy, plane_u, dx, scale_grad, stream=None):
    """The packed-plane part of linear_backward's PackedDelta branch (model.cpp:87-107):
    dx += sum_pl scales[pl] * (S_pl^T dy[t]) per row t of dy [s, rows]; scale_grad[pl] (f64,
    device) += sum(dy * plane_u[pl]). The dense dy @ W_base term is the caller's GEMM."""
    import ctypes as C

    n = len(planes)
    _req_cuda(dy, dx, scale_grad, *planes, *plane_u)
    s = dy.shape[0] if dy.dim() > 1 else 1
    if dy.shape[-1] != rows or dx.shape[-1] != cols or dx.numel() != s * cols or len(plane_u) != n \
            or len(scales) != n or scale_grad.numel() < n or any(u.numel() != s * rows for u in plane_u):
        raise BitDeltaError(8, "delta_linear_backward: length mismatch")
    bits = (C.c_void_p * max(n, 1))(*[_ptr(b) for b in planes])
    us = (C.c_void_p * max(n, 1))(*[_ptr(u.contiguous()) for u in plane_u])
    sc = (C.c_float * max(n, 1))(*[float(a) for a in scales])
    check(lib().bd_delta_linear_backward(n, bits, sc, rows, cols, _ptr(dy.contiguous()), s, us, _ptr(dx),
                                         _ptr(scale_grad), _stream(stream)))
    return dx, scale_grad


def rtn_quantize(W, stream=None):
    """rtn_quantize (int8.hpp, int8.cpp:15-42): int8 [rows, cols] values and f32 row scales,
    bit-exact with the reference. W: f32 [rows, cols] on the device."""
    import torch

    _req_cuda(W)
    w = W.contiguous()
    if w.dtype != torch.float32 or w.dim() != 2:
        raise BitDeltaError(5, "rtn_quantize: expects a 2-D f32 tensor")
    q = torch.empty(w.shape, dtype=torch.int8, device=w.device)
    sc = torch.empty(w.shape[0], dtype=torch.float32, device=w.device)
    check(lib().bd_rtn_quantize(_ptr(w), w.shape[0], w.shape[1], _ptr(q), _ptr(sc), _stream(stream)))
    return q, sc


def int8_matmul_nt(A, q, row_scales, stream=None):
    """int8_matmul_nt (int8.cpp:67-81): A [s, in] f32 times the int8 RTN tensor q [out, in]
    (row scales applied after the sum) -> [s, out] f32, on the tensor cores (kind::i8)."""
    import torch

    _req_cuda(A, q, row_scales)
    a = A.contiguous()
    if a.shape[-1] != q.shape[1] or row_scales.numel() != q.shape[0]:
        raise BitDeltaError(6, "int8_matmul_nt: inner dimensions differ")
    s = 1 if a.dim() == 1 else a.shape[0]
    y = torch.empty((s, q.shape[0]) if a.dim() > 1 else (q.shape[0],), dtype=torch.float32, device=a.device)
    check(lib().bd_int8_matmul_nt(_ptr(a), s, q.shape[1], _ptr(q.contiguous()), _ptr(row_scales.contiguous()),
                                  q.shape[0], _ptr(y), _stream(stream)))
    return y


def multitenant_linear(W, tenant_bits, tenant_alpha, req_tenant, X, stream=None):
    """Y[b] = X[b] W^T + alpha[t(b)] S_t(b) X[b]   (f32 Y).

    bf16 W/X: K2 (tcgen05) + the K3 variants; f32 W/X: K5 (SIMT, fp64 accumulation,
    the reference's own precision — BASELINE configs[0])."""
    import torch

    _req_cuda(W, X)
    if W.dtype != X.dtype or W.dtype not in (torch.bfloat16, torch.float32):
        raise BitDeltaError(5, "multitenant_linear: W and X must both be bf16 or both f32")
    out_dim, in_dim = W.shape
    B = X.shape[0]
    T = len(tenant_bits)
    bits_arr = (C.c_void_p * max(T, 1))(*[_ptr(b) for b in tenant_bits])
    alpha_arr = (C.c_float * max(T, 1))(*[float(a) for a in tenant_alpha])
    req_arr = (C.c_int32 * B)(*[int(t) for t in req_tenant])
    Y = torch.empty((B, out_dim), dtype=torch.float32, device=X.device)
    fn = lib().bd_multitenant_linear_f32 if W.dtype == torch.float32 else lib().bd_multitenant_linear
    check(fn(_ptr(W), out_dim, in_dim, T, bits_arr, alpha_arr, B, req_arr, _ptr(X), _ptr(Y), _stream(stream)))
    return Y


from .serving import ServingPool  # noqa: E402
