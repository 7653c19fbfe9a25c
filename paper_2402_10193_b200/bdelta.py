""".bdelta container (host side), the format of P:src/delta.cpp:218-334.

"BDLT", u32 LE version 1, u32 LE JSON header length, JSON array of
{name, rows, cols, kind, planes, scales, payload_offset, payload_len},
then the concatenated payloads (packed planes in the reference bit layout, or
little-endian f32 raw deltas). Entries are written in name order like the
reference's std::map, scales as the shortest decimal that round-trips the
double of the f32 (json.dump of double(float)), so files are byte-comparable.
"""
from __future__ import annotations

import json
import struct

import numpy as np

from .capi import BitDeltaError


def packed_size(rows: int, cols: int) -> int:
    return (rows * cols + 7) // 8


def read(path: str) -> dict:
    """-> {name: {kind, rows, cols, planes, scales, bits (uint8 [planes, nb]) | raw (f32 [rows, cols])}}"""
    data = open(path, "rb").read()
    if len(data) < 12:
        raise BitDeltaError(2, f"{path}: truncated .bdelta")
    if data[:4] != b"BDLT":
        raise BitDeltaError(2, f"{path}: bad magic")
    (ver,) = struct.unpack_from("<I", data, 4)
    if ver != 1:
        raise BitDeltaError(2, f"{path}: unsupported version")
    (hlen,) = struct.unpack_from("<I", data, 8)
    if hlen > len(data) - 12:
        raise BitDeltaError(2, f"{path}: header overruns file")
    try:
        header = json.loads(data[12:12 + hlen])
    except ValueError:
        raise BitDeltaError(3, f"{path}: header is not a JSON array")
    if not isinstance(header, list):
        raise BitDeltaError(3, f"{path}: header is not a JSON array")
    payload = data[12 + hlen:]
    out = {}
    for e in header:
        name = e["name"]
        if name in out:
            raise BitDeltaError(13, f"{path}: duplicate tensor '{name}'")
        rows, cols, off, ln = e["rows"], e["cols"], e["payload_offset"], e["payload_len"]
        if off > len(payload) or ln > len(payload) - off:
            raise BitDeltaError(4, f"tensor '{name}': payload out of range")
        if e["kind"] == "packed":
            planes = e["planes"]
            nb = packed_size(rows, cols)
            if ln != planes * nb:
                raise BitDeltaError(4, f"tensor '{name}': payload length does not match planes")
            scales = np.array([float(s) for s in e["scales"]], dtype=np.float32)
            if len(scales) != planes:
                raise BitDeltaError(3, f"tensor '{name}': scales/planes mismatch")
            if (scales < 0).any():
                raise BitDeltaError(9, f"tensor '{name}': negative scale")
            bits = np.frombuffer(payload, np.uint8, ln, off).reshape(planes, nb).copy()
            tail = (rows * cols) % 8
            if tail and nb and (bits[:, -1] >> tail).any():
                raise BitDeltaError(9, f"tensor '{name}': nonzero trailing bits")
            out[name] = {"kind": "packed", "rows": rows, "cols": cols, "planes": planes,
                         "scales": scales, "bits": bits}
        elif e["kind"] == "raw":
            if ln != 4 * rows * cols:
                raise BitDeltaError(4, f"tensor '{name}': payload length does not match shape")
            raw = np.frombuffer(payload, "<f4", rows * cols, off).reshape(rows, cols).copy()
            out[name] = {"kind": "raw", "rows": rows, "cols": cols, "raw": raw}
        else:
            raise BitDeltaError(3, f"tensor '{name}': unknown kind")
    return out


def _scale_json(s: np.float32) -> str:
    return json.dumps(float(np.float32(s)))


def write(delta: dict, path: str) -> None:
    """Inverse of read(); entries in name order (std::map order in the reference)."""
    parts, payload, off = [], bytearray(), 0
    for name in sorted(delta):
        e = delta[name]
        if e["kind"] == "packed":
            bits = np.ascontiguousarray(e["bits"], np.uint8).reshape(-1)
            scales = "[" + ",".join(_scale_json(s) for s in e["scales"]) + "]"
            parts.append('{"cols":%d,"kind":"packed","name":%s,"payload_len":%d,"payload_offset":%d,'
                         '"planes":%d,"rows":%d,"scales":%s}' % (e["cols"], json.dumps(name), bits.size,
                                                                  off, len(e["scales"]), e["rows"], scales))
            payload += bits.tobytes()
            off += bits.size
        else:
            raw = np.ascontiguousarray(e["raw"], "<f4").reshape(-1)
            parts.append('{"cols":%d,"kind":"raw","name":%s,"payload_len":%d,"payload_offset":%d,'
                         '"planes":0,"rows":%d,"scales":[]}' % (e["cols"], json.dumps(name), raw.size * 4,
                                                               off, e["rows"]))
            payload += raw.tobytes()
            off += raw.size * 4
    header = ("[" + ",".join(parts) + "]").encode()
    with open(path, "wb") as f:
        f.write(b"BDLT" + struct.pack("<II", 1, len(header)) + header + bytes(payload))


def entries(delta: dict) -> list[dict]:
    """Adapter for ServingPool.register_delta_entries."""
    out = []
    for name, e in delta.items():
        d = {"name": name, "kind": e["kind"], "rows": e["rows"], "cols": e["cols"]}
        if e["kind"] == "packed":
            d["bits"] = np.ascontiguousarray(e["bits"]).reshape(-1)
            d["scales"] = e["scales"]
        else:
            d["raw"] = e["raw"]
        out.append(d)
    return out
