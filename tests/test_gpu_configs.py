"""Parity on every BASELINE.json config shape through the pool's DEFAULT dispatch
(auto K3 policy, PDL, CUDA graphs) against the oracle.

The oracle for the layer stack is the C restatement (oracle/bdoracle.c, pinned
bit-for-bit to the reference ServingPool logits by tests/test_oracle.py), run on
the SAME bf16-rounded backbone with f32 activations. Per-request results of the
reference are independent of the batch composition (test_serve.cpp:169-190), so
the port runs request by request on host threads.

Shapes (P:src/arch.cpp:72-77 presets; vocab cut to 256 — the configs are about
the layer stack; embed/lm_head keep their roles):
  configs[1] Llama-2-7B layer, 8 tenants x 1 request          (byte LUT beside K2)
  configs[2] Llama-2-7B stack (2 of 32 layers), 16 x 1 and 8 x 2 at batch 16
  configs[3] Mistral-7B (GQA kv 1024, FFN 14336) at batch 64, T in {1, 16, 64}
             (K23 slots of 4 / K23 / byte LUT)
  configs[4] one Llama-2-70B layer (8192, kv 1024, FFN 28672), 32 tenants x 1
Tolerance: north star's bf16 bound, rel-L2 <= 1e-2 per request's logits (the
device path rounds GEMM activations and KV to bf16; measured values are printed).
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest
import torch

from paper_2402_10193_b200.serving import ServingPool, tensor_shapes

pytestmark = pytest.mark.gpu

PROJ = ("attn_q", "attn_k", "attn_v", "attn_o", "mlp_gate", "mlp_up", "mlp_down")


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def synth_universe(arch, n_tenants, seed, planes=lambda t: 1, alpha=2e-3):
    """bf16-exact backbone (N(0, 0.02), norms ~1) and n_tenants random deltas: packed sign
    planes for the 7 projections, raw f32 rows for norms / embed / lm_head."""
    rng = np.random.default_rng(seed)
    tens = {}
    for name, r, c in tensor_shapes(arch):
        if r == 1:
            w = 1.0 + 0.1 * rng.standard_normal((r, c), dtype=np.float32)
        else:
            w = 0.02 * rng.standard_normal((r, c), dtype=np.float32)
        tens[name] = _bf16(w)
    tenants = []
    for t in range(n_tenants):
        k = planes(t)
        ents = []
        for name, r, c in tensor_shapes(arch):
            if name.split(".")[-1] in PROJ:
                nb = (r * c + 7) // 8
                ents.append(dict(name=name, kind="packed", rows=r, cols=c,
                                 bits=rng.integers(0, 256, (k, nb), dtype=np.uint8),
                                 scales=np.array([alpha * 0.5 ** i for i in range(k)], np.float32)))
            else:
                ents.append(dict(name=name, kind="raw", rows=r, cols=c,
                                 raw=(1e-2 * rng.standard_normal((r, c), dtype=np.float32))))
        tenants.append(ents)
    return tens, tenants


def port_logits(port, arch, flat, tenants, req_tenant, tokens, pos, kc, vc, threads=16):
    """Oracle logits, one request per call (the reference's per-request independence)."""
    port_ents = [[dict(e, raw=e["raw"].reshape(-1)) if e["kind"] == "raw" else e for e in es]
                 for es in tenants]

    def one(i):
        return port.decode(arch, flat, [port_ents[req_tenant[i]]], [0], [tokens[i]], [pos[i]],
                           [kc[i]], [vc[i]])[0]

    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        return np.stack(list(ex.map(one, range(len(req_tenant)))))


def run_config(port, arch, n_tenants, batch, steps=2, seed=0, planes=lambda t: 1, expect_paths=None,
               int8=False):
    """int8: the INT8 RTN backbone (ServingPool(QuantizedCheckpoint), serve.cpp:99-108): the 7
    projections quantized by the reference rule (port.rtn_quantize, bit-exact with the
    device's), the oracle run on rtn_dequantize (int8.cpp:44-53) of the same values."""
    arch = dict(arch, vocab=256, max_seq=8, rope_theta=10000.0)
    tens, tenants = synth_universe(arch, n_tenants, seed, planes)
    if int8:
        for name in list(tens):
            if name.split(".")[-1] in PROJ:
                q, sc = port.rtn_quantize(tens[name])
                tens[name] = (q, sc)
    pool = ServingPool(arch, tens)
    if int8:
        for name in list(tens):
            if isinstance(tens[name], tuple):
                q, sc = tens[name]
                tens[name] = q.astype(np.float32) * sc[:, None]
    for t, ents in enumerate(tenants):
        pool.register_delta_entries(f"t{t}", ents)
    req_tenant = [b % n_tenants for b in range(batch)]  # round robin (serve.cpp:410)
    rids = [pool.open_request(f"t{t}") for t in req_tenant]
    flat = np.concatenate([tens[n].reshape(-1) for n, _, _ in tensor_shapes(arch)])
    del tens
    kc = [np.zeros((arch["n_layers"], arch["max_seq"], arch["kv_dim"]), np.float32) for _ in range(batch)]
    vc = [np.zeros_like(k) for k in kc]
    rng = np.random.default_rng(seed + 1)
    worst = 0.0
    for pos in range(steps):
        toks = [int(t) for t in rng.integers(0, arch["vocab"], batch)]
        got = pool.decode_step([(r, toks[i], pos) for i, r in enumerate(rids)])
        if expect_paths is not None:
            assert pool.stats()["delta_paths"] == expect_paths, pool.stats()["delta_paths"]
        want = port_logits(port, arch, flat, tenants, req_tenant, toks, [pos] * batch, kc, vc)
        errs = [rel_l2(got[i], want[i]) for i in range(batch)]
        worst = max(worst, max(errs))
    pool.close()
    print(f"max rel-L2 over {batch} requests x {steps} steps: {worst:.3e}")
    return worst


L7 = dict(dim=4096, kv_dim=4096, n_heads=32, intermediate=11008)
M7 = dict(dim=4096, kv_dim=1024, n_heads=32, intermediate=14336)
L70 = dict(dim=8192, kv_dim=1024, n_heads=64, intermediate=28672)


def test_config1_l7_layer_T8_B8(cuda, port):
    assert run_config(port, dict(L7, n_layers=1), 8, 8, steps=3, expect_paths="LLLL") <= 1e-2


@pytest.mark.parametrize("tenants", [16, 8])
def test_config2_l7_stack_B16(cuda, port, tenants):
    """configs[2] at batch 16 (2 of the 32 layers): 16 x 1 request and 8 x 2 requests."""
    assert run_config(port, dict(L7, n_layers=2), tenants, 16, steps=2, seed=tenants,
                      expect_paths="LLLL") <= 1e-2


@pytest.mark.parametrize("tenants,paths", [(1, "DDDD"), (4, "DDDD"), (8, "DDDD"), (16, "TTTT"), (64, "LLLL")])
def test_config3_m7_gqa_B64(cuda, port, tenants, paths):
    """configs[3]: Mistral-7B GQA (kv_dim 1024 < dim), batch 64, tenant sweep through the
    default dispatch (K3d from 8 requests per tenant, K23 from 2, the byte LUT below)."""
    assert run_config(port, dict(M7, n_layers=1), tenants, 64, steps=2, seed=100 + tenants,
                      expect_paths=paths) <= 1e-2


def test_config3_k23_one_tenant_B64(cuda, port, monkeypatch):
    """K23 (slots of 4 requests) kept under test at one tenant x 64 requests (forced)."""
    monkeypatch.setenv("BD_DELTA", "mt4")
    assert run_config(port, dict(M7, n_layers=1), 1, 64, steps=2, seed=101, expect_paths="TTTT") <= 1e-2


def test_config4_l70_layer_T32_B32(cuda, port):
    """configs[4]: one Llama-2-70B layer (GQA, 8192 / 28672), 32 tenants x 1 request."""
    assert run_config(port, dict(L70, n_layers=1), 32, 32, steps=2, seed=70, expect_paths="LLLL") <= 1e-2


@pytest.mark.parametrize("planes,tenants,batch", [((2, 3), 4, 4), ((2, 3), 2, 8)])
def test_multi_plane_stacks_default_paths(cuda, port, planes, tenants, batch):
    """k = 2 and 3 plane stacks (compress_stack, delta.cpp:57-70; serve.cpp:22-26) through the
    byte LUT (1 request per tenant) and K23 (4 per tenant) on a 128-multiple shape."""
    arch = dict(dim=512, kv_dim=512, n_heads=4, intermediate=1024, n_layers=2)
    paths = "LLLL" if batch == tenants else "TTTT"
    assert run_config(port, arch, tenants, batch, steps=3, seed=5, planes=lambda t: planes[t % 2],
                      expect_paths=paths) <= 1e-2


def test_int8_backbone_l7_layer_T8_B8(cuda, port):
    """the configs[1] layer on an INT8 RTN backbone (K2 kind::i8 beside the
    byte LUT) against the oracle on the dequantized backbone."""
    assert run_config(port, dict(L7, n_layers=1), 8, 8, steps=3, expect_paths="LLLL", int8=True) <= 1e-2


def test_int8_backbone_m7_gqa_B64_T16(cuda, port):
    """int8 backbone at batch 64 (256 MMA columns of pieces), GQA, 4 requests per tenant: the
    LUT (K23 fuses a bf16 GEMM and is not planned for an int8 backbone)."""
    assert run_config(port, dict(M7, n_layers=1), 16, 64, steps=1, expect_paths="LLLL", int8=True) <= 1e-2


@pytest.mark.parametrize("arch,n_layers,tenants,batch", [
    (M7, 1, 1, 64),     # configs[3] T=1: one tenant, 64 requests (N = 64)
    (M7, 1, 4, 64),     # configs[3] T=4: 16 requests per tenant
    (L7, 2, 3, 40),     # 14/13/13 requests: N padded to 16, 2 layers
])
def test_k3d_many_requests_per_tenant(cuda, port, monkeypatch, arch, n_layers, tenants, batch):
    """K3d (mtd.cu): a tenant's plane expanded once to bf16 +-1 in TMEM and applied to all
    of its requests as the N of a kind::f16 MMA, against the oracle."""
    monkeypatch.setenv("BD_DELTA", "mtd")
    assert run_config(port, dict(arch, n_layers=n_layers), tenants, batch, steps=2, expect_paths="DDDD") <= 1e-2
