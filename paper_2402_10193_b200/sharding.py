"""Output-row sharding of the BitDelta layer stack over `world` GPUs.

Mirrors PoolImpl::local_rows / run_layers (csrc/pool.cu): rank r of W owns rows
[r*R/W, (r+1)*R/W) of every projection and of each tenant's packed planes. With
cols % 8 == 0 a row shard of a plane is the contiguous byte range
[r0*cols/8, (r0+nr)*cols/8) of the reference layout, so shards are sliced
straight out of the .bdelta bytes. q/k/v rows are whole heads, so attention is
local; per layer four all-gathers (ctx, o-out, act, down-out) rebuild the full
vectors, concatenated in rank order.
"""
from __future__ import annotations

from typing import Mapping

PROJ = ("attn_q", "attn_k", "attn_v", "attn_o", "mlp_gate", "mlp_up", "mlp_down")


def check(arch: Mapping, world: int) -> None:
    dim, kv, heads = arch["dim"], arch.get("kv_dim", arch["dim"]), arch["n_heads"]
    hd = dim // heads
    n_kv = kv // hd
    if n_kv % world or arch["intermediate"] % world:
        raise ValueError("kv heads and intermediate must divide by the world size")


def local_rows(arch: Mapping, role: str, world: int, rank: int) -> tuple[int, int]:
    """(first row, row count) of this rank's shard of projection `role`."""
    dim, kv, inter = arch["dim"], arch.get("kv_dim", arch["dim"]), arch["intermediate"]
    rows = {"attn_q": dim, "attn_k": kv, "attn_v": kv, "attn_o": dim, "mlp_gate": inter,
            "mlp_up": inter, "mlp_down": dim}[role]
    n = rows // world
    return rank * n, n


def plane_bytes(r0: int, nr: int, cols: int) -> tuple[int, int]:
    """Byte range of rows [r0, r0+nr) in a packed plane (flat LSB-first layout)."""
    if (r0 * cols) % 8 or (nr * cols) % 8:
        raise ValueError("row shard does not start/end on a byte of the packed plane")
    return r0 * cols // 8, (r0 + nr) * cols // 8


def gathered_to_full(parts):
    """All-gather result (list over ranks of [B, n_l]) -> [B, W*n_l] in rank column order."""
    import numpy as np

    return np.concatenate(parts, axis=1)
