"""GPU parity of the kernels behind the C-ABI (K1 compress, K3 packed apply,
K2+K3 multi-tenant linear) against the oracle / golden vectors from the
reference. Bit-exact for bits; tolerances stated per test."""
import os

import numpy as np
import pytest
import torch

import paper_2402_10193_b200 as bd

pytestmark = pytest.mark.gpu


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return np.linalg.norm(got - want) / (den if den > 0 else 1.0)


def torch_pack(delta: torch.Tensor) -> torch.Tensor:
    """Independent packer (flat LSB-first) used for size-independent checks."""
    v = (delta.reshape(-1) > 0).to(torch.uint8)
    n = v.numel()
    pad = (-n) % 8
    if pad:
        v = torch.cat([v, torch.zeros(pad, dtype=torch.uint8, device=v.device)])
    w = torch.tensor([1, 2, 4, 8, 16, 32, 64, 128], dtype=torch.int32, device=v.device)
    return (v.view(-1, 8).to(torch.int32) * w).sum(1).to(torch.uint8)


def test_compress_golden_f32(cuda, golden):
    exact_alpha = 0
    n = int(golden["n_cases"])
    for i in range(n):
        base = torch.from_numpy(golden[f"c{i}_base"]).to(cuda)
        fine = torch.from_numpy(golden[f"c{i}_fine"]).to(cuda)
        bits, alpha = bd.compress_tensor(base, fine)
        assert np.array_equal(bits.cpu().numpy(), golden[f"c{i}_bits"]), i
        a, want = alpha.item(), float(golden[f"c{i}_scale"])
        assert abs(a - want) <= 1e-5 * abs(want) + 1e-30, (i, a, want)  # north star: 1e-5 rel
        exact_alpha += np.float32(a).view(np.uint32) == np.float32(want).view(np.uint32)
    assert exact_alpha == n  # fp64 accumulation: bit-identical on every golden case


def test_compress_kats(cuda, golden):
    bits, alpha = bd.compress_delta(torch.tensor([[1, -1, 1], [1, -1, -1], [1, -1, 1]], dtype=torch.float32, device=cuda))
    assert bits.tolist() == [0x4D, 0x01] and alpha.item() == 1.0
    # sign rule: 0, -0, NaN, tiny values (test_delta.cpp:24-30)
    v = torch.from_numpy(golden["kat_sign_in"]).to(cuda).view(1, -1)
    bits, _ = bd.compress_delta(v)
    got = [(int(bits[i // 8]) >> (i % 8)) & 1 for i in range(v.numel())]
    assert [1 if s == 1 else 0 for s in golden["kat_sign_out"]] == got
    z = torch.randn(6, 5, device=cuda)
    bits, alpha = bd.compress_tensor(z, z)
    assert alpha.item() == 0.0 and int(bits.sum()) == 0


def test_compress_bf16_and_ragged(cuda, port):
    g = torch.Generator(device="cpu").manual_seed(1)
    for rows, cols in [(1, 1), (3, 5), (7, 9), (33, 65), (128, 4096), (17, 1000)]:
        base = (torch.randn(rows, cols, generator=g) * 0.02).to(torch.bfloat16)
        fine = (base.float() + torch.randn(rows, cols, generator=g) * 1e-3).to(torch.bfloat16)
        bits, alpha = bd.compress_tensor(base.to(cuda), fine.to(cuda))
        wb, wa = port.compress_tensor(base.float().numpy(), fine.float().numpy())
        assert np.array_equal(bits.cpu().numpy(), wb), (rows, cols)
        assert abs(alpha.item() - wa) <= 1e-6 * wa


@pytest.mark.parametrize("shape", [(4096, 4096), (11008, 4096), (4096, 11008)])
def test_compress_full_size_properties(cuda, shape):
    torch.manual_seed(0)
    base = (torch.randn(shape, device=cuda) * 0.02).to(torch.bfloat16)
    fine = (base.float() + torch.randn(shape, device=cuda) * 1e-3).to(torch.bfloat16)
    bits, alpha = bd.compress_tensor(base, fine)
    d = fine.float() - base.float()
    assert torch.equal(bits, torch_pack(d))
    want = d.double().abs().sum().item() / d.numel()
    assert abs(alpha.item() - want) <= 1e-6 * want
    # idempotence: compress(decompress(p)) keeps the bits (test_delta.cpp:89-92)
    signs = torch.where(d > 0, 1.0, -1.0) * alpha.item()
    b2, a2 = bd.compress_delta(signs)
    assert torch.equal(b2, bits) and abs(a2.item() - alpha.item()) <= 1e-6 * alpha.item()


def test_compress_batched_matches_single(cuda):
    torch.manual_seed(2)
    pairs = []
    for rows, cols in [(64, 64), (100, 37), (4096, 1024), (1, 9), (1024, 11008)]:
        b = torch.randn(rows, cols, device=cuda)
        pairs.append((b, b + 0.01 * torch.randn(rows, cols, device=cuda)))
    outs = bd.compress_batched(pairs)
    for (b, f), (bits, alpha) in zip(pairs, outs):
        b1, a1 = bd.compress_tensor(b, f)
        assert torch.equal(bits, b1) and alpha.item() == a1.item()


def test_compress_stack_golden(cuda, golden):
    for i in range(int(golden["n_cases"])):
        base = torch.from_numpy(golden[f"c{i}_base"]).to(cuda)
        fine = torch.from_numpy(golden[f"c{i}_fine"]).to(cuda)
        bits, alphas = bd.compress_stack(base, fine, 3)
        wb, ws = golden[f"c{i}_stack_bits"], golden[f"c{i}_stack_scales"]
        assert np.array_equal(bits[0].cpu().numpy(), wb[0]), i
        # every plane bit-exact: plane k fits the residual left by planes < k, which is
        # bit-identical as long as each alpha is (fp64 accumulation: bit-identical here)
        assert np.array_equal(bits.cpu().numpy(), wb), i
        assert np.array_equal(alphas.cpu().numpy().view(np.uint32), ws.view(np.uint32)), (i, alphas, ws)


def test_packed_signed_accumulate_golden(cuda, golden):
    for i in range(int(golden["n_cases"])):
        bits = torch.from_numpy(golden[f"c{i}_bits"]).to(cuda)
        rows, cols = golden[f"c{i}_base"].shape
        x = torch.from_numpy(golden[f"c{i}_x"]).to(cuda)
        out = torch.from_numpy(golden[f"c{i}_out0"]).to(cuda).clone()
        bd.packed_signed_accumulate(bits, rows, cols, x, out)
        want = golden[f"c{i}_acc"]
        assert rel_l2(out.cpu().numpy(), want) <= 1e-6, i  # a7: fp64 accumulation like the reference
        assert (out.cpu().numpy() == want).mean() > 0.95


def test_packed_matvec_kats_and_random(cuda, port):
    b1, _ = bd.compress_delta(torch.ones(1, 3, device=cuda))
    assert bd.packed_matvec(b1, 1.0, 1, 3, torch.tensor([1.0, 2, 3], device=cuda)).item() == 6.0
    b2, _ = bd.compress_delta(torch.tensor([[1.0, -1.0]], device=cuda))
    assert bd.packed_matvec(b2, 2.0, 1, 2, torch.tensor([3.0, 1.0], device=cuda)).item() == 4.0
    rng = np.random.default_rng(5)
    for _ in range(30):  # acceptance.cpp:121-131: random 1..96 dims vs dense oracle
        rows, cols = int(rng.integers(1, 97)), int(rng.integers(1, 97))
        d = rng.standard_normal((rows, cols)).astype(np.float32)
        x = rng.standard_normal(cols).astype(np.float32)
        bits, alpha = bd.compress_delta(torch.from_numpy(d).to(cuda))
        got = bd.packed_matvec(bits, alpha.item(), rows, cols, torch.from_numpy(x).to(cuda)).cpu().numpy()
        dense = port.decompress(bits.cpu().numpy(), rows, cols, alpha.item())
        want = (dense.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)
        assert rel_l2(got, want) <= 1e-5


def test_packed_accumulate_large_linearity(cuda):
    torch.manual_seed(3)
    rows, cols = 4096, 11008
    d = torch.randn(rows, cols, device=cuda)
    bits, _ = bd.compress_delta(d)
    x = torch.randn(2, cols, device=cuda)
    out = torch.zeros(2, rows, device=cuda)
    bd.packed_signed_accumulate(bits, rows, cols, x, out)
    S = torch.where(d > 0, 1.0, -1.0).double()
    want = (x.double() @ S.T)
    assert rel_l2(out.cpu().numpy(), want.cpu().numpy()) <= 1e-6
    # linearity (test_delta.cpp:189-209)
    o2 = torch.zeros(1, rows, device=cuda)
    bd.packed_signed_accumulate(bits, rows, cols, (x[0] + x[1]).view(1, -1), o2)
    assert rel_l2(o2[0].cpu().numpy(), (out[0] + out[1]).cpu().numpy()) <= 1e-5


def _mt_reference(W, bits_list, alphas, req_tenant, X, rows, cols):
    Wd, Xd = W.double(), X.double()
    Y = Xd @ Wd.T
    for b, t in enumerate(req_tenant):
        if t < 0:
            continue
        v = torch.tensor([1, 2, 4, 8, 16, 32, 64, 128], dtype=torch.uint8, device=W.device)
        unpacked = ((bits_list[t].view(-1, 1) & v) != 0).view(-1)[: rows * cols].view(rows, cols)
        S = torch.where(unpacked, 1.0, -1.0).double()
        Y[b] += alphas[t] * (S @ Xd[b])
    return Y


@pytest.mark.parametrize("rows,cols,B,T", [(4096, 4096, 16, 16), (11008, 4096, 8, 8), (4096, 11008, 16, 4),
                                           (200, 64, 5, 3), (1024, 4096, 64, 1), (384, 1024, 1, 1)])
def test_multitenant_linear(cuda, rows, cols, B, T):
    torch.manual_seed(rows + cols + B)
    W = (torch.randn(rows, cols, device=cuda) * 0.02).to(torch.bfloat16)
    X = torch.randn(B, cols, device=cuda).to(torch.bfloat16)
    bits_list, alphas = [], []
    for t in range(T):
        fine = (W.float() + torch.randn(rows, cols, device=cuda) * 1e-3).to(torch.bfloat16)
        b, a = bd.compress_tensor(W, fine)
        bits_list.append(b)
        alphas.append(a.item())
    req_tenant = [b % T for b in range(B)]
    if B > 2:
        req_tenant[-1] = -1  # a base-only request
    Y = bd.multitenant_linear(W, bits_list, alphas, req_tenant, X)
    want = _mt_reference(W, bits_list, alphas, req_tenant, X, rows, cols)
    # bf16 operands are exact; only f32 accumulation order differs
    assert rel_l2(Y.cpu().numpy(), want.cpu().numpy()) <= 1e-5


def _delta_only_case(rows, cols, B, T, cuda):
    torch.manual_seed(7 + rows)
    W = torch.zeros(rows, cols, device=cuda, dtype=torch.bfloat16)
    # activations with a wide dynamic range inside each 32-column block
    X = (torch.randn(B, cols, device=cuda) * torch.exp(2 * torch.randn(B, cols, device=cuda))).to(torch.bfloat16)
    bits_list, alphas = [], []
    for t in range(T):
        b, a = bd.compress_tensor(torch.zeros(rows, cols, device=cuda), torch.randn(rows, cols, device=cuda))
        bits_list.append(b)
        alphas.append(a.item())
    rt = [b % T for b in range(B)]
    Y = bd.multitenant_linear(W, bits_list, alphas, rt, X)
    want = _mt_reference(W, bits_list, alphas, rt, X, rows, cols)
    return rel_l2(Y.cpu().numpy(), want.cpu().numpy())


@pytest.mark.parametrize("rows,cols,B,T", [(4096, 4096, 16, 16), (1024, 11008, 8, 3), (512, 1024, 1, 1)])
def test_multitenant_linear_delta_only(cuda, rows, cols, B, T):
    """Zero backbone: Y is the delta term alone, so its error is not diluted by the base
    product (default path) — within 1e-5 rel-L2 of f64."""
    assert _delta_only_case(rows, cols, B, T, cuda) <= 1e-5


@pytest.mark.parametrize("mode", ["mt4", "lut", "units"])
def test_multitenant_linear_delta_only_each_path(cuda, mode):
    """Delta term alone through K23 (FP4 pieces, ~1e-7 measured), the byte LUT and the
    SIMT units."""
    import subprocess
    import sys

    code = f"""
import sys; sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))})
sys.path.insert(0, {repr(os.path.dirname(os.path.abspath(__file__)))})
import torch
from test_gpu_kernels import _delta_only_case
dev = torch.device('cuda:0')
for case in [(4096, 4096, 16, 16), (1024, 11008, 8, 3), (512, 1024, 1, 1), (1024, 4096, 64, 4)]:
    err = _delta_only_case(*case, dev)
    assert err <= 1e-5, (case, err)
print('ok')
"""
    env = dict(os.environ, BD_DELTA=mode)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_multitenant_linear_permutation_bit_identical(cuda):
    torch.manual_seed(9)
    rows, cols, B, T = 1024, 2048, 12, 5
    W = (torch.randn(rows, cols, device=cuda) * 0.02).to(torch.bfloat16)
    X = torch.randn(B, cols, device=cuda).to(torch.bfloat16)
    bits_list, alphas = [], []
    for t in range(T):
        b, a = bd.compress_tensor(W, (W.float() + 1e-3 * torch.randn_like(W.float())).to(torch.bfloat16))
        bits_list.append(b)
        alphas.append(a.item())
    rt = [b % T for b in range(B)]
    Y = bd.multitenant_linear(W, bits_list, alphas, rt, X)
    perm = list(reversed(range(B)))
    Yp = bd.multitenant_linear(W, bits_list, alphas, [rt[p] for p in perm], X[perm].contiguous())
    assert torch.equal(Yp, Y[perm])


@pytest.mark.parametrize("mode", ["mt4", "lut", "units"])
def test_multitenant_linear_each_delta_path(cuda, mode):
    """Every K3 variant (K23 FP4 tensor cores, byte-LUT, SIMT units) against the same f64 reference."""
    import subprocess
    import sys

    code = f"""
import sys; sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))})
sys.path.insert(0, {repr(os.path.dirname(os.path.abspath(__file__)))})
import torch, numpy as np
import paper_2402_10193_b200 as bd
from test_gpu_kernels import _mt_reference, rel_l2
dev = torch.device('cuda:0')
for rows, cols, B, T in [(4096, 4096, 16, 16), (768, 11008, 8, 2), (1024, 2048, 12, 3)]:
    torch.manual_seed(rows + B)
    W = (torch.randn(rows, cols, device=dev) * 0.02).to(torch.bfloat16)
    X = torch.randn(B, cols, device=dev).to(torch.bfloat16)
    bits, al = [], []
    for t in range(T):
        b, a = bd.compress_tensor(W, (W.float() + 1e-3 * torch.randn_like(W.float())).to(torch.bfloat16))
        bits.append(b); al.append(a.item())
    rt = [b % T for b in range(B)]
    Y = bd.multitenant_linear(W, bits, al, rt, X)
    err = rel_l2(Y.cpu().numpy(), _mt_reference(W, bits, al, rt, X, rows, cols).cpu().numpy())
    assert err <= 1e-5, (rows, cols, B, T, err)
print('ok')
"""
    env = dict(os.environ, BD_DELTA=mode)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_config0_compress_4096sq_f32_vs_reference(cuda, ref):
    """BASELINE configs[0]: one 4096x4096 fp32 base + fine-tune pair compressed on the GPU,
    bits bit-exact and alpha within 1e-5 (bit-identical here) of the reference library."""
    rng = np.random.default_rng(4096)
    base = (rng.standard_normal((4096, 4096), dtype=np.float32) * 0.02)
    fine = (base + rng.standard_normal((4096, 4096), dtype=np.float32) * 1e-3).astype(np.float32)
    bits, alpha = bd.compress_tensor(torch.from_numpy(base).to(cuda), torch.from_numpy(fine).to(cuda))
    wb, wa = ref.compress_tensor(base, fine)
    assert np.array_equal(bits.cpu().numpy(), wb)
    assert abs(alpha.item() - wa) <= 1e-5 * wa
    assert np.float32(alpha.item()).view(np.uint32) == np.float32(wa).view(np.uint32)


def test_config0_apply_f32_batch4_vs_reference(cuda, ref):
    """BASELINE configs[0] apply step in the reference's f32: 4 tenants (tenant 0 = the
    compressed pair), one request each, Y = W x + alpha S x through K5 vs the reference's
    matmul_nt + packed_matvec; rel-L2 <= 1e-5 (north star f32 tolerance)."""
    rng = np.random.default_rng(40960)
    n = 4096
    W = rng.standard_normal((n, n), dtype=np.float32) * 0.02
    X = rng.standard_normal((4, n), dtype=np.float32)
    bits, alphas = [], []
    for t in range(4):
        fine = (W + rng.standard_normal((n, n), dtype=np.float32) * 1e-3).astype(np.float32)
        b, a = ref.compress_tensor(W, fine)
        bits.append(b)
        alphas.append(float(a))
    Wd = torch.from_numpy(W).to(cuda)
    Y = bd.multitenant_linear(Wd, [torch.from_numpy(b).to(cuda) for b in bits], alphas, [0, 1, 2, 3],
                              torch.from_numpy(X).to(cuda)).cpu().numpy()
    base = ref.matmul_nt(X, W)
    for b in range(4):
        want = base[b] + ref.packed_matvec(bits[b], n, n, alphas[b], X[b])
        assert rel_l2(Y[b], want) <= 1e-5, (b, rel_l2(Y[b], want))


def test_config4_compress_l70_mlp_shape_vs_reference(cuda, ref):
    """K1 at the largest BASELINE shape (Llama-2-70B mlp_gate 28672 x 8192, bf16 inputs as the
    bench compresses them) against the reference library: bits bit-exact, alpha <= 1e-5."""
    g = torch.Generator(device="cuda").manual_seed(70)
    shape = (28672, 8192)
    base = (torch.randn(shape, device=cuda, generator=g) * 0.02).to(torch.bfloat16)
    fine = (base.float() + torch.randn(shape, device=cuda, generator=g) * 1e-3).to(torch.bfloat16)
    bits, alpha = bd.compress_tensor(base, fine)
    wb, wa = ref.compress_tensor(base.float().cpu().numpy(), fine.float().cpu().numpy())
    assert np.array_equal(bits.cpu().numpy(), wb)
    assert abs(alpha.item() - wa) <= 1e-5 * wa
