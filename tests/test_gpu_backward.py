"""GPU parity of K6, the distillation backward pieces:
packed_signed_accumulate_t (P:src/delta.cpp:105-131) and linear_backward's
PackedDelta branch (P:src/model.cpp:87-107: dx += alpha * S^T dy, alpha grad
= sum dy * u), against the reference (golden fixtures made by oracle/_ref, and
the reference live where it is built)."""
import os

import numpy as np
import pytest
import torch

import paper_2402_10193_b200 as bd
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return np.linalg.norm(got - want) / (den if den > 0 else 1.0)


def test_transpose_accumulate_golden(cuda):
    """Every golden case (ragged shapes, zero y entries, accumulation onto a nonzero out,
    3 vectors per launch) within 1e-6 relative L2 of the reference (fp64 column sums like
    the reference; only the summation order differs), and mostly bit-identical."""
    g = np.load(os.path.join(GOLDEN, "backward_v1.npz"))
    same = total = 0
    for i in range(int(g["n_cases"])):
        rows, cols = (int(v) for v in g[f"t{i}_shape"])
        bits = torch.from_numpy(g[f"t{i}_bits"]).to(cuda)
        y = torch.from_numpy(g[f"t{i}_y"]).to(cuda)
        out = torch.from_numpy(g[f"t{i}_out0"]).to(cuda)
        bd.packed_signed_accumulate_t(bits, rows, cols, y, out)
        got, want = out.cpu().numpy(), g[f"t{i}_out"]
        assert rel_l2(got, want) <= 1e-6, i
        same += int((got == want).sum())
        total += want.size
    assert same >= 0.99 * total, (same, total)


@pytest.mark.parametrize("rows,cols", [(4096, 4096), (11008, 4096), (4096, 11008), (1000, 777)])
def test_transpose_accumulate_vs_reference_large(cuda, ref, rows, cols):
    rng = np.random.default_rng(rows + cols)
    d = rng.standard_normal((rows, cols)).astype(np.float32)
    bits, _ = ref.compress_delta(d)
    y = rng.standard_normal((2, rows)).astype(np.float32)
    want = np.stack([ref.packed_signed_accumulate_t(bits, rows, cols, y[v]) for v in range(2)])
    out = torch.zeros(2, cols, device=cuda)
    bd.packed_signed_accumulate_t(torch.from_numpy(bits).to(cuda), rows, cols, torch.from_numpy(y).to(cuda), out)
    assert rel_l2(out.cpu().numpy(), want) <= 1e-6


def test_transpose_is_adjoint_of_forward(cuda):
    """<S x, y> == <x, S^T y> through the two drop-ins (size-independent property)."""
    g = torch.Generator(device="cpu").manual_seed(5)
    rows, cols = 3000, 2048
    d = torch.randn(rows, cols, generator=g).to(cuda)
    bits, _ = bd.compress_delta(d)
    x = torch.randn(cols, generator=g).to(cuda)
    y = torch.randn(rows, generator=g).to(cuda)
    sx = torch.zeros(rows, device=cuda)
    sty = torch.zeros(cols, device=cuda)
    bd.packed_signed_accumulate(bits, rows, cols, x, sx)
    bd.packed_signed_accumulate_t(bits, rows, cols, y, sty)
    a = float(torch.dot(sx.double(), y.double()))
    b = float(torch.dot(x.double(), sty.double()))
    assert abs(a - b) <= 1e-5 * (abs(a) + 1.0)


def test_delta_linear_backward_vs_reference(cuda, ref):
    """linear_backward's PackedDelta branch (model.cpp:87-107) for a 2-plane linear,
    s = 5 rows of dy: dx accumulation and the fp64 alpha gradients against the reference's
    own pieces composed exactly as model.cpp does (per plane: g = sum double(dy)*u;
    col = packed_signed_accumulate_t(plane, dy[t]); dx[t] += s * col)."""
    rng = np.random.default_rng(3)
    rows, cols, s = 384, 520, 5
    base = rng.standard_normal((rows, cols)).astype(np.float32)
    fine = base + 0.05 * rng.standard_normal((rows, cols)).astype(np.float32)
    pbits, pscales = ref.compress_stack(base, fine, 2)
    x = rng.standard_normal((s, cols)).astype(np.float32)
    dy = rng.standard_normal((s, rows)).astype(np.float32)
    dx0 = rng.standard_normal((s, cols)).astype(np.float32)
    us = [np.stack([ref.packed_signed_accumulate(pbits[pl], rows, cols, x[t]) for t in range(s)]) for pl in range(2)]
    want_dx = dx0.copy()
    want_g = np.zeros(2)
    for pl in range(2):
        want_g[pl] += float(np.sum(dy.astype(np.float64) * us[pl].astype(np.float64)))
        for t in range(s):
            col = ref.packed_signed_accumulate_t(pbits[pl], rows, cols, dy[t])
            want_dx[t] = want_dx[t] + np.float32(pscales[pl]) * col
    dx = torch.from_numpy(dx0).to(cuda)
    sg = torch.zeros(2, dtype=torch.float64, device=cuda)
    planes = [torch.from_numpy(pbits[pl]).to(cuda) for pl in range(2)]
    bd.delta_linear_backward(planes, [float(v) for v in pscales], rows, cols, torch.from_numpy(dy).to(cuda),
                             [torch.from_numpy(u).to(cuda) for u in us], dx, sg)
    assert rel_l2(dx.cpu().numpy(), want_dx) <= 1e-6
    np.testing.assert_allclose(sg.cpu().numpy(), want_g, rtol=1e-12)
