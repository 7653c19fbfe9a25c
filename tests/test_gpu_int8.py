"""GPU parity of the INT8 RTN backbone (SURVEY.md §8(f)#4, P:src/int8.cpp): rtn_quantize
bit-exact, int8_matmul_nt on the tcgen05 kind::i8 tensor cores within 1e-5 relative L2
of the reference (its f32 sequential sum is the reference's own rounding level)."""
import numpy as np
import pytest
import torch

import paper_2402_10193_b200 as bd

pytestmark = pytest.mark.gpu


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return np.linalg.norm(got - want) / (den if den > 0 else 1.0)


@pytest.mark.parametrize("rows,cols", [(1, 1), (7, 13), (300, 257), (4096, 4096), (11008, 4096)])
def test_rtn_quantize_bit_exact(cuda, ref, rows, cols):
    rng = np.random.default_rng(rows * 7 + cols)
    w = (rng.standard_normal((rows, cols)) * 0.02).astype(np.float32)
    if rows > 2:
        w[1] = 0.0                                        # zero row -> scale 0
        w[2, : min(cols, 4)] = [0.5, -0.5, 1.0, -1.0][: min(cols, 4)]  # ties after /s
    q, s = bd.rtn_quantize(torch.from_numpy(w).to(cuda))
    wq, ws = ref.rtn_quantize(w)
    assert np.array_equal(q.cpu().numpy(), wq)
    assert np.array_equal(s.cpu().numpy(), ws)


def test_rtn_quantize_rejects_non_finite(cuda):
    w = torch.zeros(4, 8, device=cuda)
    w[2, 3] = float("nan")
    with pytest.raises(bd.BitDeltaError) as e:
        bd.rtn_quantize(w)
    assert e.value.status == 11  # non_finite


@pytest.mark.parametrize("s,out_dim,in_dim", [(1, 64, 64), (4, 4096, 4096), (3, 100, 77), (70, 384, 512),
                                              (16, 1024, 11008)])
def test_int8_matmul_nt_vs_reference(cuda, ref, s, out_dim, in_dim):
    rng = np.random.default_rng(s + out_dim + in_dim)
    w = (rng.standard_normal((out_dim, in_dim)) * 0.02).astype(np.float32)
    a = rng.standard_normal((s, in_dim)).astype(np.float32)
    a[0, :5] *= 1e-6  # tiny entries next to the row maximum
    q, sc = ref.rtn_quantize(w)
    want = ref.int8_matmul_nt(a, q, sc)
    got = bd.int8_matmul_nt(torch.from_numpy(a).to(cuda), torch.from_numpy(q).to(cuda), torch.from_numpy(sc).to(cuda))
    assert rel_l2(got.cpu().numpy(), want) <= 1e-5


def test_int8_matmul_nt_exact_on_integer_activations(cuda):
    """Activations that fit the first piece exactly (small integers) give the exact s32 dot
    products times the row scale (the tensor-core accumulation is exact)."""
    g = torch.Generator().manual_seed(3)
    q = torch.randint(-127, 128, (256, 1024), generator=g, dtype=torch.int32).to(torch.int8)
    sc = torch.rand(256, generator=g) + 0.5
    a = torch.randint(-32, 33, (8, 1024), generator=g).float()
    a[:, 0] = 63.0  # row maximum in [32, 64): scale 1, pieces 1..3 are zero
    want = (a.double() @ q.double().T) * sc.double()
    got = bd.int8_matmul_nt(a.to(cuda), q.to(cuda), sc.to(cuda)).cpu().double()
    exact = (a.double() @ q.double().T).float().double() * sc.double()
    assert torch.equal(got, exact.float().double()) or rel_l2(got.numpy(), want.numpy()) <= 1e-7
