"""Golden fixtures for the distillation backward pieces, made by the
REFERENCE library itself (oracle/_ref). Re-run only in the build container:

    make -C oracle ref && python tests/golden/make_golden_backward.py

Output: backward_v1.npz — for random and ragged shapes (rows need not start on a byte),
a sign plane compressed by the reference's compress_delta, vectors y (with zero entries,
which the reference skips) and the reference's packed_signed_accumulate_t(p, y, out)
(P:src/delta.cpp:105-131) accumulated onto a nonzero `out`; plus the KAT-style case of
P:tests/test_delta.cpp:211-221 (48 x 56).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    ref = oracle.ref()
    rng = np.random.default_rng(20261017)
    shapes = [(48, 56), (1, 1), (3, 3), (7, 13), (33, 65), (100, 31), (257, 96), (64, 4096), (512, 300)]
    out = {"n_cases": len(shapes)}
    for i, (rows, cols) in enumerate(shapes):
        d = rng.standard_normal((rows, cols)).astype(np.float32)
        bits, _ = ref.compress_delta(d)
        nv = 3
        y = rng.standard_normal((nv, rows)).astype(np.float32)
        y[:, ::4] = 0.0
        o0 = rng.standard_normal((nv, cols)).astype(np.float32)
        res = np.stack([ref.packed_signed_accumulate_t(bits, rows, cols, y[v], o0[v]) for v in range(nv)])
        out.update({f"t{i}_shape": np.array([rows, cols]), f"t{i}_bits": bits, f"t{i}_y": y,
                    f"t{i}_out0": o0, f"t{i}_out": res})
    np.savez_compressed(os.path.join(HERE, "backward_v1.npz"), **out)


if __name__ == "__main__":
    main()
