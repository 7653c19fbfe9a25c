"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
library itself (oracle/_ref/libdeltakit_ref.so, built from /root/reference by
oracle/Makefile). Re-run only in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed, small):
  golden_v1.npz         KATs from P:tests/test_delta.cpp + random-shape compress /
                        packed_signed_accumulate / matmul_nt outputs of the reference
  toy_*.bdelta          4 tenant deltas written by the reference's write_delta_file
                        for the test_serve.cpp universe (kCfg, seeds 1001 / 2000+i)
  toy_decode.npz        backbone (synth_base), token streams and the reference
                        ServingPool shared-mode logits for B in {1,2,4}
  mp_t*.bdelta, mp_decode.npz (--mp)  2- and 3-plane deltas on a 256-dim config
                        written by the reference, and its logits for B in {4,16}
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

# P:tests/test_serve.cpp:16-17
TOY_CFG = {"vocab": 48, "dim": 32, "n_layers": 2, "n_heads": 4, "intermediate": 40, "max_seq": 32,
           "rope_theta": 10000.0}


def main():
    r = oracle.ref()
    rng = np.random.default_rng(20240215)
    g = {}
    # --- KATs (P:tests/test_delta.cpp) ---
    g["kat_sign_in"] = np.array([3.2, 0.0, -0.0, -1e-30, 1e-30, np.nan, np.inf, -np.inf, 1.4e-45],
                                np.float32)
    g["kat_sign_out"] = np.array([r.sign_of(float(v)) for v in g["kat_sign_in"]], np.int32)
    bits, s = r.compress_tensor(np.zeros((2, 2), np.float32), np.array([[1, -2], [3, -4]], np.float32))
    g["kat_2x2_bits"], g["kat_2x2_scale"] = bits, np.float32(s)
    bits, s = r.compress_delta(np.array([[1, -1, 1], [1, -1, -1], [1, -1, 1]], np.float32))
    g["kat_3x3_bits"], g["kat_3x3_scale"] = bits, np.float32(s)  # 0x4D, 0x01
    p1 = r.packed_matvec(r.compress_delta(np.ones((1, 3), np.float32))[0], 1, 3, 1.0, np.array([1, 2, 3], np.float32))
    p2 = r.packed_matvec(r.compress_delta(np.array([[1, -1]], np.float32))[0], 1, 2, 2.0, np.array([3, 1], np.float32))
    g["kat_matvec"] = np.array([p1[0], p2[0]], np.float32)  # 6, 4

    # --- random shapes (ragged, 1..96 like acceptance.cpp:121-131, plus larger) ---
    shapes = [(1, 1), (1, 7), (3, 3), (5, 9), (7, 13), (9, 21), (12, 23), (17, 33), (31, 64),
              (64, 64), (96, 95), (40, 172), (128, 256), (255, 77), (300, 40)]
    for i, (rows, cols) in enumerate(shapes):
        base = (rng.standard_normal((rows, cols)) * 0.02).astype(np.float32)
        fine = (base + rng.standard_normal((rows, cols)) * 1e-3).astype(np.float32)
        if i % 5 == 0:  # exact zeros and signed zeros in the delta
            fine.flat[:: 3] = base.flat[:: 3]
        bits, s = r.compress_tensor(base, fine)
        x = rng.standard_normal((2, cols)).astype(np.float32)
        out0 = rng.standard_normal((2, rows)).astype(np.float32)
        acc = np.stack([r.packed_signed_accumulate(bits, rows, cols, x[v], out0[v]) for v in range(2)])
        g[f"c{i}_base"], g[f"c{i}_fine"], g[f"c{i}_bits"], g[f"c{i}_scale"] = base, fine, bits, np.float32(s)
        g[f"c{i}_x"], g[f"c{i}_out0"], g[f"c{i}_acc"] = x, out0, acc
        sb, ss = r.compress_stack(base, fine, 3)
        g[f"c{i}_stack_bits"], g[f"c{i}_stack_scales"] = sb, ss
    g["n_cases"] = np.int32(len(shapes))
    a = rng.standard_normal((4, 96)).astype(np.float32)
    w = rng.standard_normal((50, 96)).astype(np.float32)
    g["mm_a"], g["mm_w"], g["mm_out"] = a, w, r.matmul_nt(a, w)
    np.savez_compressed(os.path.join(HERE, "golden_v1.npz"), **g)

    # --- toy serving universe (P:tests/test_serve.cpp:19-45) ---
    cfg = json.dumps({k: v for k, v in TOY_CFG.items()})
    base = r.synth_base(cfg, 1001, 0.08)
    for i in range(4):
        fine = r.synth_fine(cfg, base, 0.03, 2000 + i)
        r.write_delta_file(cfg, base, fine, 1, os.path.join(HERE, f"toy_t{i}.bdelta"))
    zero_path = os.path.join(HERE, "toy_zero.bdelta")
    r.write_delta_file(cfg, base, base, 1, zero_path)
    d = {"cfg": np.array(cfg), "base": base}
    for B in (1, 2, 4):
        pool = r.pool(cfg, base)
        for i in range(min(B, 4)):
            pool.register_delta(f"t{i}", os.path.join(HERE, f"toy_t{i}.bdelta"))
        rids = [pool.open_request(f"t{i % 4}") for i in range(B)]
        stream = np.random.default_rng(42 + B).integers(0, TOY_CFG["vocab"], 6).astype(np.int32)
        logits = []
        for pos, tok in enumerate(stream):
            logits.append(pool.decode_step([(rid, int(tok), pos) for rid in rids]))
        d[f"B{B}_tokens"] = stream
        d[f"B{B}_logits"] = np.stack(logits)  # [steps, B, vocab]
    np.savez_compressed(os.path.join(HERE, "toy_decode.npz"), **d)
    # raw little-endian copies for the C++ shim test (tests/cpp/test_deltakit_gpu.cpp)
    base.astype("<f4").tofile(os.path.join(HERE, "toy_base.f32"))
    d["B4_tokens"].astype("<i4").tofile(os.path.join(HERE, "toy_tokens_B4.i32"))
    d["B4_logits"].astype("<f4").tofile(os.path.join(HERE, "toy_logits_B4.f32"))
    print("golden fixtures written to", HERE)


# multi-plane universe on a 128-multiple shape (the byte-LUT / K23 paths; the toy above
# only reaches the SIMT units): tenants with 2 and 3 sign planes per projection
# (compress_stack, P:src/delta.cpp:57-70; --bits k of P:tools/main.cpp:455-460)
MP_CFG = {"vocab": 64, "dim": 256, "n_layers": 1, "n_heads": 2, "intermediate": 512, "max_seq": 16,
          "rope_theta": 10000.0}
MP_PLANES = [2, 3, 3, 2]


def mp_universe():
    r = oracle.ref()
    cfg = json.dumps(MP_CFG)
    base = r.synth_base(cfg, 3003, 0.08)
    for i, k in enumerate(MP_PLANES):
        fine = r.synth_fine(cfg, base, 0.03, 4000 + i)
        r.write_delta_file(cfg, base, fine, k, os.path.join(HERE, f"mp_t{i}.bdelta"))
    d = {"cfg": np.array(cfg), "base": base}
    # B = 4: one request per tenant; B = 16: four per tenant (the K23 slots)
    for B in (4, 16):
        pool = r.pool(cfg, base)
        for i in range(len(MP_PLANES)):
            pool.register_delta(f"t{i}", os.path.join(HERE, f"mp_t{i}.bdelta"))
        rids = [pool.open_request(f"t{i % len(MP_PLANES)}") for i in range(B)]
        stream = np.random.default_rng(77 + B).integers(0, MP_CFG["vocab"], 4).astype(np.int32)
        logits = [pool.decode_step([(rid, int(tok), pos) for rid in rids]) for pos, tok in enumerate(stream)]
        d[f"B{B}_tokens"] = stream
        d[f"B{B}_logits"] = np.stack(logits)
    np.savez_compressed(os.path.join(HERE, "mp_decode.npz"), **d)
    print("multi-plane fixtures written to", HERE)


if __name__ == "__main__":
    if "--mp" in sys.argv:
        mp_universe()
    else:
        main()
