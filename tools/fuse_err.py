"""Fused vs separate step epilogues (BD_EPI_FUSE) on the reference-written multi-plane
.bdelta case of tests/test_gpu_pool.py: max rel-L2 of the logits vs the reference (experiments)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from conftest import GOLDEN  # noqa: E402
from paper_2402_10193_b200.serving import ServingPool, tensor_shapes  # noqa: E402


def tensors_of(arch, flat):
    out, o = {}, 0
    for n, r, c in tensor_shapes(arch):
        out[n] = flat[o:o + r * c].reshape(r, c)
        o += r * c
    return out


d = np.load(os.path.join(GOLDEN, "mp_decode.npz"))
arch = dict(json.loads(str(d["cfg"])))
arch["kv_dim"] = arch["dim"]
for fz in ("1", "0"):
    os.environ["BD_EPI_FUSE"] = fz
    for B in (4, 16):
        pool = ServingPool(arch, tensors_of(arch, d["base"]))
        for i in range(4):
            pool.register_delta(f"t{i}", os.path.join(GOLDEN, f"mp_t{i}.bdelta"))
        rids = [pool.open_request(f"t{i % 4}") for i in range(B)]
        errs = []
        for pos, tok in enumerate(d[f"B{B}_tokens"]):
            got = pool.decode_step([(r, int(tok), pos) for r in rids])
            want = d[f"B{B}_logits"][pos]
            errs.append(max(np.linalg.norm(got[i] - want[i]) / np.linalg.norm(want[i]) for i in range(B)))
        print(f"fuse={fz} B={B} paths={pool.stats()['delta_paths']} max_err_per_pos={np.round(errs, 5).tolist()}")
        pool.close()
