"""ServingPool — Python mirror of deltakit::ServingPool (P:include/deltakit/serve.hpp:59-100)
over the device-resident pool in libbitdelta_b200.so (bd_pool_* in capi.h)."""
from __future__ import annotations

import ctypes as C
from typing import Iterable, Mapping

import numpy as np

from .capi import BD_BF16, BD_F32, Arch, DeltaEntry, PoolStats, Request, check, lib

SHARED, NAIVE = "shared", "naive"  # ServeMode (serve.hpp:18)
# default_quantize_policy (P:src/delta.cpp:150-161): the 7 layer projections
PROJECTIONS = ("attn_q", "attn_k", "attn_v", "attn_o", "mlp_gate", "mlp_up", "mlp_down")


def tensor_shapes(arch: Mapping) -> list[tuple[str, int, int]]:
    """tensor_shapes (P:src/arch.cpp:51-69) with kv_dim for k/v (preset_shapes, arch.cpp:92-110)."""
    dim, kv, inter, vocab = arch["dim"], arch.get("kv_dim", arch["dim"]), arch["intermediate"], arch["vocab"]
    out = [("embed", vocab, dim)]
    for i in range(arch["n_layers"]):
        p = f"layers.{i}."
        out += [(p + "attn_q", dim, dim), (p + "attn_k", kv, dim), (p + "attn_v", kv, dim),
                (p + "attn_o", dim, dim), (p + "mlp_gate", inter, dim), (p + "mlp_up", inter, dim),
                (p + "mlp_down", dim, inter), (p + "norm1", 1, dim), (p + "norm2", 1, dim)]
    out += [("final_norm", 1, dim), ("lm_head", vocab, dim)]
    return out


class ServingPool:
    """One resident backbone on one GPU (or one row shard of it), N registered
    deltas, per-request bf16 KV caches. decode_step(mode="shared") runs one
    backbone pass per step for the whole batch (serve.cpp:205-325)."""

    def __init__(self, arch: Mapping, tensors: Mapping | None = None, device: int = 0,
                 world_size: int = 1, rank: int = 0, int8: bool = False):
        """int8=True: ServingPool(QuantizedCheckpoint) (serve.cpp:99-108) built like
        rtn_quantize_checkpoint(base, default_quantize_policy()) — the 7 layer projections
        RTN-quantized on the device (bd_rtn_quantize), everything else dense. A tensor given
        as a (int8 values, f32 row scales) pair is taken as already quantized."""
        self.arch = dict(arch)
        self.arch.setdefault("kv_dim", self.arch["dim"])
        self.arch.setdefault("rope_theta", 10000.0)
        check(lib().bd_device_check(device))
        a = Arch(self.arch["vocab"], self.arch["dim"], self.arch["kv_dim"], self.arch["n_layers"],
                 self.arch["n_heads"], self.arch["intermediate"], self.arch["max_seq"],
                 float(self.arch["rope_theta"]))
        h = C.c_void_p()
        check(lib().bd_pool_create(C.byref(a), device, world_size, rank, C.byref(h)))
        self._h = h
        self.device = device
        self._ids: list[str] = []
        if tensors is not None:
            for name, t in tensors.items():
                if isinstance(t, tuple):
                    self.set_tensor_i8(name, *t)
                elif int8 and name.split(".")[-1] in PROJECTIONS:
                    self.set_tensor_i8(name, *self._rtn(t))
                else:
                    self.set_tensor(name, t)

    def _rtn(self, data):
        import torch

        from . import rtn_quantize

        t = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data, np.float32))
        return rtn_quantize(t.float().to(f"cuda:{self.device}"))

    def set_tensor_i8(self, name: str, q, row_scales) -> None:
        """One projection as an Int8Tensor (int8.hpp): int8 [rows, cols] + f32 [rows]."""
        import torch

        if isinstance(q, torch.Tensor):
            qq, ss = q.contiguous(), row_scales.float().contiguous()
            check(lib().bd_pool_set_tensor_i8(self._h, name.encode(), qq.data_ptr(), ss.data_ptr(), int(qq.is_cuda),
                                              qq.shape[0], qq.shape[1]))
        else:
            qq = np.ascontiguousarray(q, np.int8)
            ss = np.ascontiguousarray(row_scales, np.float32)
            check(lib().bd_pool_set_tensor_i8(self._h, name.encode(), qq.ctypes.data, ss.ctypes.data, 0,
                                              qq.shape[0], qq.shape[1]))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().bd_pool_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    # ---- multi-GPU (row-sharded pool, world_size > 1) ----
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().bd_nccl_unique_id(buf))
        return buf.raw

    def init_comm(self, uid: bytes) -> None:
        """Every rank, after rank 0's nccl_unique_id() was broadcast."""
        buf = C.create_string_buffer(uid, 128)
        check(lib().bd_pool_init_comm(self._h, buf))

    def init_loopback(self, group: str) -> None:
        """Test hook: the row-sharded pools of one process on one device exchange by device
        copies instead of NCCL (drive each rank's decode from its own thread)."""
        check(lib().bd_pool_init_loopback(self._h, group.encode()))

    # ---- backbone ----
    def set_tensor(self, name: str, data) -> None:
        import torch

        if isinstance(data, torch.Tensor):
            t = data.contiguous()
            if t.dim() == 1:
                t = t.view(1, -1)
            dt = BD_BF16 if t.dtype == torch.bfloat16 else BD_F32
            if t.dtype not in (torch.bfloat16, torch.float32):
                t = t.float()
                dt = BD_F32
            check(lib().bd_pool_set_tensor(self._h, name.encode(), t.data_ptr(), dt, int(t.is_cuda),
                                           t.shape[0], t.shape[1]))
        else:
            a = np.ascontiguousarray(data, dtype=np.float32)
            if a.ndim == 1:
                a = a.reshape(1, -1)
            check(lib().bd_pool_set_tensor(self._h, name.encode(), a.ctypes.data, BD_F32, 0,
                                           a.shape[0], a.shape[1]))

    # ---- tenants (serve.hpp:64-66) ----
    def register_delta(self, id_: str, path: str, resident: bool = True) -> None:
        check(lib().bd_pool_register_delta_file(self._h, id_.encode(), str(path).encode(), int(resident)))
        self._ids.append(id_)

    def register_delta_entries(self, id_: str, entries: Iterable[Mapping]) -> None:
        """entries: {name, kind: 'packed'|'raw', rows, cols, bits (np.uint8 [planes*nb] or
        cuda uint8 tensor), scales (floats), raw (np.float32 or cuda tensor)}"""
        import torch

        ents = list(entries)
        arr = (DeltaEntry * len(ents))()
        keep = []
        for i, e in enumerate(ents):
            name = e["name"].encode()
            keep.append(name)
            if e["kind"] == "packed":
                scales = np.ascontiguousarray(e["scales"], np.float32)
                sc = (C.c_float * len(scales))(*scales.tolist())
                keep.append(sc)
                bits = e["bits"]
                if isinstance(bits, torch.Tensor):
                    ptr, dev = bits.data_ptr(), int(bits.is_cuda)
                    keep.append(bits)
                else:
                    b = np.ascontiguousarray(bits, np.uint8)
                    keep.append(b)
                    ptr, dev = b.ctypes.data, 0
                arr[i] = DeltaEntry(name, 1, e["rows"], e["cols"], len(scales), ptr, sc, None, dev)
            else:
                raw = e["raw"]
                if raw is None:  # all-zero raw delta (nothing resident)
                    arr[i] = DeltaEntry(name, 0, e["rows"], e["cols"], 0, None, None, None, 0)
                    continue
                if isinstance(raw, torch.Tensor):
                    r = raw.contiguous().float()
                    keep.append(r)
                    ptr, dev = r.data_ptr(), int(r.is_cuda)
                else:
                    r = np.ascontiguousarray(raw, np.float32)
                    keep.append(r)
                    ptr, dev = r.ctypes.data, 0
                arr[i] = DeltaEntry(name, 0, e["rows"], e["cols"], 0, None, None, ptr, dev)
        check(lib().bd_pool_register_delta(self._h, id_.encode(), arr, len(ents)))
        self._ids.append(id_)

    def delta_ids(self) -> list[str]:
        return sorted(self._ids)

    # ---- requests ----
    def open_request(self, delta_id: str) -> int:
        r = C.c_uint64()
        check(lib().bd_pool_open_request(self._h, delta_id.encode(), C.byref(r)))
        return r.value

    def close_request(self, request_id: int) -> None:
        check(lib().bd_pool_close_request(self._h, request_id))

    @staticmethod
    def _batch(reqs):
        arr = (Request * len(reqs))()
        for i, (rid, tok, pos) in enumerate(reqs):
            arr[i] = Request(rid, tok, pos)
        return arr

    def decode_step(self, reqs, mode: str = SHARED) -> np.ndarray:
        """reqs: [(request_id, token, position)] -> logits f32 [B, vocab] (serve.hpp:70)."""
        import torch

        n = len(reqs)
        out = np.zeros((n, self.arch["vocab"]), np.float32)
        s = torch.cuda.current_stream(self.device).cuda_stream
        check(lib().bd_pool_decode_step(self._h, self._batch(reqs), n, 0 if mode == SHARED else 1,
                                        out.ctypes.data, s))
        return out

    def decode_layers(self, reqs, x_in, x_out=None, stream=None):
        """The layer stack only, on device-resident activations (f32 [B, dim])."""
        import torch

        if x_out is None:
            x_out = torch.empty_like(x_in)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check(lib().bd_pool_decode_layers(self._h, self._batch(reqs), len(reqs), x_in.data_ptr(),
                                          x_out.data_ptr(), s))
        return x_out

    def stats(self) -> dict:
        st = PoolStats()
        check(lib().bd_pool_get_stats(self._h, C.byref(st)))
        return {"backbone_passes": st.backbone_passes, "cold_loads": st.cold_loads,
                "last_cold_load_ms": st.last_cold_load_ms, "resident_bytes": st.resident_bytes,
                "kernels_last_step": st.kernels_last_step, "delta_paths": st.delta_paths.decode()}

    def resident_bytes(self) -> int:
        return self.stats()["resident_bytes"]
