"""GPU ServingPool (bd_pool_*) parity with the reference ServingPool
(P:tests/test_serve.cpp, acceptance.cpp criterion 3) and the oracle port.

Tolerances: the device pool computes in bf16 (weights, GEMM activations, KV)
with f32 accumulation, so logits are compared with relative L2 <= 1e-2 against
the f32 reference (north star's bf16 tolerance), and <= 5e-3 against the port
run on the same bf16-rounded backbone. Determinism / permutation / counters
are exact."""
import json
import os

import numpy as np
import pytest
import torch

import paper_2402_10193_b200 as bd
from conftest import GOLDEN
from paper_2402_10193_b200 import bdelta
from paper_2402_10193_b200.serving import ServingPool, tensor_shapes

pytestmark = pytest.mark.gpu


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)


def bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


@pytest.fixture(scope="module")
def toy():
    d = np.load(os.path.join(GOLDEN, "toy_decode.npz"))
    cfg = json.loads(str(d["cfg"]))
    arch = dict(cfg, kv_dim=cfg["dim"])
    return d, arch


def tensors_of(arch, flat):
    out, off = {}, 0
    for name, r, c in tensor_shapes(arch):
        out[name] = flat[off:off + r * c].reshape(r, c)
        off += r * c
    return out


def make_pool(cuda, arch, base, n_tenants=4, resident=True):
    pool = ServingPool(arch, tensors_of(arch, base))
    for i in range(n_tenants):
        pool.register_delta(f"t{i}", os.path.join(GOLDEN, f"toy_t{i}.bdelta"), resident)
    return pool


def test_shared_matches_reference_logits(cuda, toy):
    """acceptance.cpp:133-173 / test_serve.cpp:103-132 against the golden reference logits."""
    d, arch = toy
    for B in (1, 2, 4):
        pool = make_pool(cuda, arch, d["base"])
        rids = [pool.open_request(f"t{i % 4}") for i in range(B)]
        for pos, tok in enumerate(d[f"B{B}_tokens"]):
            got = pool.decode_step([(r, int(tok), pos) for r in rids])
            want = d[f"B{B}_logits"][pos]
            for i in range(B):
                assert rel_l2(got[i], want[i]) <= 1e-2, (B, pos, i, rel_l2(got[i], want[i]))
        pool.close()


def test_shared_matches_port_on_bf16_backbone(cuda, toy, port):
    d, arch = toy
    base16 = bf16_round(d["base"])
    names = [n for n, _, _ in tensor_shapes(arch)]
    tens = [[bdelta.read(os.path.join(GOLDEN, f"toy_t{i}.bdelta"))[n] for n in names] for i in range(4)]
    B = 4
    pool = make_pool(cuda, arch, base16)
    rids = [pool.open_request(f"t{i}") for i in range(B)]
    kc = [np.zeros((arch["n_layers"], arch["max_seq"], arch["kv_dim"]), np.float32) for _ in range(B)]
    vc = [np.zeros_like(k) for k in kc]
    toks = d["B4_tokens"]
    for pos, tok in enumerate(toks):
        got = pool.decode_step([(r, int(tok), pos) for r in rids])
        want = port.decode(arch, base16, tens, list(range(B)), [int(tok)] * B, [pos] * B, kc, vc)
        for i in range(B):
            assert rel_l2(got[i], want[i]) <= 5e-3, (pos, i, rel_l2(got[i], want[i]))


def test_identical_contexts_identical_outputs(cuda, toy):
    """test_serve.cpp:134-145"""
    d, arch = toy
    pool = make_pool(cuda, arch, d["base"], 1)
    a, b = pool.open_request("t0"), pool.open_request("t0")
    out = pool.decode_step([(a, 7, 0), (b, 7, 0)])
    assert np.array_equal(out[0], out[1])


def test_permutation_bit_identical(cuda, toy):
    """test_serve.cpp:169-190"""
    d, arch = toy

    def run(order):
        pool = make_pool(cuda, arch, d["base"], 3)
        reqs = [pool.open_request(f"t{i}") for i in range(3)]
        out = None
        for pos in range(2):
            out = pool.decode_step([(reqs[i], 5 + i, pos) for i in order])
        return out

    fwd, rev = run([0, 1, 2]), run([2, 1, 0])
    for i in range(3):
        assert np.array_equal(fwd[i], rev[2 - i])


def test_zero_delta_equals_backbone(cuda, toy, port):
    """test_serve.cpp:147-167: a zero delta decodes like the plain backbone."""
    d, arch = toy
    base16 = bf16_round(d["base"])
    pool = ServingPool(arch, tensors_of(arch, base16))
    pool.register_delta("zero", os.path.join(GOLDEN, "toy_zero.bdelta"))
    r = pool.open_request("zero")
    names = [n for n, _, _ in tensor_shapes(arch)]
    zero = [bdelta.read(os.path.join(GOLDEN, "toy_zero.bdelta"))[n] for n in names]
    kc = [np.zeros((arch["n_layers"], arch["max_seq"], arch["kv_dim"]), np.float32)]
    vc = [np.zeros_like(kc[0])]
    for pos, tok in enumerate([3, 11, 40, 2, 9]):
        got = pool.decode_step([(r, tok, pos)])[0]
        want = port.decode(arch, base16, [zero], [0], [tok], [pos], kc, vc)[0]
        assert rel_l2(got, want) <= 5e-3


def test_backbone_pass_counter(cuda, toy):
    """test_serve.cpp:192-210"""
    d, arch = toy
    pool = make_pool(cuda, arch, d["base"])
    reqs = [pool.open_request(f"t{i}") for i in range(4)]
    pool.decode_step([(r, 1, 0) for r in reqs])
    assert pool.stats()["backbone_passes"] == 1
    pool.decode_step([(r, 1, 1) for r in reqs])
    assert pool.stats()["backbone_passes"] == 2
    pool.decode_step([(r, 1, 2) for r in reqs], mode="naive")
    assert pool.stats()["backbone_passes"] == 2 + 4


def test_naive_matches_shared(cuda, toy):
    d, arch = toy
    ps, pn = make_pool(cuda, arch, d["base"]), make_pool(cuda, arch, d["base"])
    rs = [ps.open_request(f"t{i}") for i in range(4)]
    rn = [pn.open_request(f"t{i}") for i in range(4)]
    for pos, tok in enumerate([1, 2, 3]):
        zs = ps.decode_step([(r, tok, pos) for r in rs])
        zn = pn.decode_step([(r, tok, pos) for r in rn], mode="naive")
        for i in range(4):
            assert rel_l2(zs[i], zn[i]) <= 1e-4


def test_cold_registration_hot_swap(cuda, toy):
    """test_serve.cpp:62-76"""
    d, arch = toy
    pool = ServingPool(arch, tensors_of(arch, d["base"]))
    before = pool.resident_bytes()
    pool.register_delta("cold", os.path.join(GOLDEN, "toy_t0.bdelta"), resident=False)
    assert pool.resident_bytes() == before and pool.stats()["cold_loads"] == 0
    r = pool.open_request("cold")
    pool.decode_step([(r, 3, 0)])
    st = pool.stats()
    assert st["cold_loads"] == 1 and st["last_cold_load_ms"] > 0
    assert pool.resident_bytes() > before


def test_registration_and_decode_errors(cuda, toy, tmp_path):
    d, arch = toy
    pool = make_pool(cuda, arch, d["base"], 1)
    with pytest.raises(bd.BitDeltaError) as e:
        pool.register_delta("t0", os.path.join(GOLDEN, "toy_t0.bdelta"))
    assert e.value.code == "duplicate_id"
    # wrong-arch delta names the first offending tensor (test_serve.cpp:78-100)
    f = bdelta.read(os.path.join(GOLDEN, "toy_t0.bdelta"))
    f["embed"] = {"kind": "raw", "rows": 2, "cols": 2, "raw": np.zeros((2, 2), np.float32)}
    p = str(tmp_path / "bad.bdelta")
    bdelta.write(f, p)
    with pytest.raises(bd.BitDeltaError) as e:
        pool.register_delta("bad", p)
    assert e.value.code == "shape_mismatch" and "'embed'" in str(e.value)
    r = pool.open_request("t0")
    with pytest.raises(bd.BitDeltaError) as e:
        pool.decode_step([(r, 10_000, 0)])
    assert e.value.code == "bad_token"
    with pytest.raises(bd.BitDeltaError) as e:
        pool.decode_step([(r, 1, 3)])
    assert e.value.code == "bad_argument"
    with pytest.raises(bd.BitDeltaError) as e:
        pool.decode_step([(99, 1, 0)])
    assert e.value.code == "unknown_id"
    with pytest.raises(bd.BitDeltaError) as e:
        pool.open_request("nope")
    assert e.value.code == "unknown_id"


def test_memory_accounting(cuda, toy):
    """test_serve.cpp:212-241: resident = backbone + delta payloads + caches."""
    d, arch = toy
    pool = make_pool(cuda, arch, d["base"], 2)
    backbone = sum(4 * r * c for _, r, c in tensor_shapes(arch))
    payload = 0
    for i in range(2):
        for e in bdelta.read(os.path.join(GOLDEN, f"toy_t{i}.bdelta")).values():
            payload += e["planes"] * (e["bits"].shape[1] + 4) if e["kind"] == "packed" else 4 * e["raw"].size
    assert pool.resident_bytes() == backbone + payload
    r0, r1 = pool.open_request("t0"), pool.open_request("t1")
    for pos in range(3):
        pool.decode_step([(r0, 1, pos), (r1, 2, pos)])
    kv = 2 * 2 * 4 * 3 * arch["dim"] * arch["n_layers"]
    assert pool.resident_bytes() == backbone + payload + kv


def test_cpp_mirror_program(cuda):
    """The deltakit_gpu C++ mirror (include/deltakit_gpu) passes its re-hosted reference cases."""
    import subprocess

    from conftest import ROOT

    exe = os.path.join(ROOT, "tests", "cpp", "test_deltakit_gpu")
    if not os.path.exists(exe):
        from paper_2402_10193_b200 import build

        build.build()
    r = subprocess.run([exe, GOLDEN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr


def _random_entries(arch, rng, alpha=2e-3, raw_sigma=1e-2):
    ents = []
    for name, r, c in tensor_shapes(arch):
        if r > 1 and name != "embed" and name != "lm_head":
            nb = (r * c + 7) // 8
            ents.append(dict(name=name, kind="packed", rows=r, cols=c,
                             bits=rng.integers(0, 256, (1, nb), dtype=np.uint8),
                             scales=np.array([alpha], np.float32)))
        else:
            ents.append(dict(name=name, kind="raw", rows=r, cols=c,
                             raw=(rng.standard_normal((r, c)) * raw_sigma).astype(np.float32)))
    return ents


@pytest.mark.parametrize("dim,n_heads,kv_dim", [(256, 2, 256), (512, 4, 256), (1024, 8, 256), (1024, 8, 128)])
def test_head_dim_128_long_context_matches_port(cuda, port, dim, n_heads, kv_dim):
    """The head_dim-128 attention kernels past their 192-row shared-memory staging (two K/V
    chunks), two tenants, against the port on a bf16 backbone: multi-head (the Llama-2-7B
    shape) and grouped-query with 2, 4 and 8 query heads per KV head (attn128g_kernel: one
    CTA per request and KV head; Mistral-7B has 4, Llama-2-70B 8)."""
    arch = dict(vocab=64, dim=dim, n_layers=1, n_heads=n_heads, intermediate=512, max_seq=220,
                rope_theta=10000.0, kv_dim=kv_dim)
    rng = np.random.default_rng(7)
    tens = {}
    for name, r, c in tensor_shapes(arch):
        w = rng.standard_normal((r, c)).astype(np.float32) * (1.0 if r == 1 else 0.05)
        tens[name] = bf16_round(w + (1.0 if r == 1 else 0.0))
    pool = ServingPool(arch, tens)
    ents = [_random_entries(arch, rng) for _ in range(2)]
    for t, e in enumerate(ents):
        pool.register_delta_entries(f"t{t}", e)
    rids = [pool.open_request(f"t{t}") for t in range(2)]
    names = [n for n, _, _ in tensor_shapes(arch)]
    port_ents = [[{k: v for k, v in e.items()} for e in es] for es in ents]
    for es in port_ents:
        for e in es:
            if e["kind"] == "raw":
                e["raw"] = e["raw"].reshape(-1)
    flat = np.concatenate([tens[n].reshape(-1) for n in names])
    kc = [np.zeros((1, arch["max_seq"], arch["kv_dim"]), np.float32) for _ in range(2)]
    vc = [np.zeros_like(k) for k in kc]
    toks = rng.integers(0, arch["vocab"], 200)
    for pos, tok in enumerate(toks):
        got = pool.decode_step([(r, int(tok), pos) for r in rids])
        want = port.decode(arch, flat, port_ents, [0, 1], [int(tok)] * 2, [pos] * 2, kc, vc)
        if pos % 16 == 0 or pos >= 188:
            for i in range(2):
                # bf16 activations/KV against the f32 port: 4e-3..1.3e-2 measured here,
                # identical with the generic attention kernel (BD_ATTN_OLD=1)
                err = rel_l2(got[i], want[i])
                assert err <= 2e-2, (pos, i, err)
    pool.close()


def test_gqa_long_max_seq_uses_per_head_attention(cuda, port):
    """Grouped-query heads whose G score buffers do not fit in shared memory (8 query heads per
    KV head at max_seq 7000) fall back to one CTA per query head instead of failing."""
    arch = dict(vocab=64, dim=1024, n_layers=1, n_heads=8, intermediate=512, max_seq=7000,
                rope_theta=10000.0, kv_dim=128)
    rng = np.random.default_rng(11)
    tens = {}
    for name, r, c in tensor_shapes(arch):
        w = rng.standard_normal((r, c)).astype(np.float32) * (1.0 if r == 1 else 0.05)
        tens[name] = bf16_round(w + (1.0 if r == 1 else 0.0))
    pool = ServingPool(arch, tens)
    ents = [_random_entries(arch, rng) for _ in range(2)]
    for t, e in enumerate(ents):
        pool.register_delta_entries(f"t{t}", e)
    rids = [pool.open_request(f"t{t}") for t in range(2)]
    names = [n for n, _, _ in tensor_shapes(arch)]
    port_ents = [[{k: v for k, v in e.items()} for e in es] for es in ents]
    for es in port_ents:
        for e in es:
            if e["kind"] == "raw":
                e["raw"] = e["raw"].reshape(-1)
    flat = np.concatenate([tens[n].reshape(-1) for n in names])
    kc = [np.zeros((1, arch["max_seq"], arch["kv_dim"]), np.float32) for _ in range(2)]
    vc = [np.zeros_like(k) for k in kc]
    for pos, tok in enumerate(rng.integers(0, arch["vocab"], 4)):
        got = pool.decode_step([(r, int(tok), pos) for r in rids])
        want = port.decode(arch, flat, port_ents, [0, 1], [int(tok)] * 2, [pos] * 2, kc, vc)
        for i in range(2):
            assert rel_l2(got[i], want[i]) <= 2e-2, (pos, i, rel_l2(got[i], want[i]))
    pool.close()


def _k23_pool_run(port, B_per_t, steps, n_tenants=2, dim=256, inter=512, n_layers=2):
    """n_tenants tenants x B_per_t requests each on a 128-multiple shape (K23-eligible),
    several decode steps against the port on the same bf16 backbone."""
    arch = dict(vocab=64, dim=dim, n_layers=n_layers, n_heads=dim // 128, intermediate=inter, max_seq=16,
                rope_theta=10000.0, kv_dim=dim)
    rng = np.random.default_rng(11)
    tens = {}
    for name, r, c in tensor_shapes(arch):
        w = rng.standard_normal((r, c)).astype(np.float32) * (1.0 if r == 1 else 0.05)
        tens[name] = bf16_round(w + (1.0 if r == 1 else 0.0))
    pool = ServingPool(arch, tens)
    ents = [_random_entries(arch, rng) for _ in range(n_tenants)]
    for t, e in enumerate(ents):
        pool.register_delta_entries(f"t{t}", e)
    B = n_tenants * B_per_t
    rids = [pool.open_request(f"t{b % n_tenants}") for b in range(B)]
    names = [n for n, _, _ in tensor_shapes(arch)]
    port_ents = [[{k: v for k, v in e.items()} for e in es] for es in ents]
    for es in port_ents:
        for e in es:
            if e["kind"] == "raw":
                e["raw"] = e["raw"].reshape(-1)
    flat = np.concatenate([tens[n].reshape(-1) for n in names])
    kc = [np.zeros((arch["n_layers"], arch["max_seq"], arch["kv_dim"]), np.float32) for _ in range(B)]
    vc = [np.zeros_like(k) for k in kc]
    errs = []
    for pos in range(steps):
        toks = [int(t) for t in rng.integers(0, arch["vocab"], B)]
        got = pool.decode_step([(r, toks[i], pos) for i, r in enumerate(rids)])
        want = port.decode(arch, flat, port_ents, [b % n_tenants for b in range(B)], toks, [pos] * B, kc, vc)
        errs.append(max(rel_l2(got[i], want[i]) for i in range(B)))
    pool.close()
    return max(errs)


def test_k23_pool_many_requests_per_tenant(cuda, port):
    """Six requests per tenant: the pool's default picks K23 (base GEMM + FP4 tensor-core
    deltas in one kernel); logits against the port within the bf16 tolerance."""
    assert _k23_pool_run(port, 6, 4) <= 1e-2


def test_k23_pool_forced_one_request_per_tenant(cuda, port):
    import subprocess
    import sys

    code = f"""
import sys; sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))})
sys.path.insert(0, {repr(os.path.dirname(os.path.abspath(__file__)))})
import oracle
from test_gpu_pool import _k23_pool_run
err = _k23_pool_run(oracle.port(), 1, 4)
assert err <= 1e-2, err
print('ok')
"""
    env = dict(os.environ, BD_DELTA="mt4")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_k23_pool_two_request_slots_short_plane_ring(cuda, port):
    """K23 with 2-request slots on one Llama-2-7B-shaped layer (8 tenants x 2 requests): the
    plane-stage ring is then as short as the producer count, the case whose mbarrier phases
    aliased (launch failure) before the per-slot fill guard (mt4.cu); logits against the port."""
    import subprocess
    import sys

    code = f"""
import sys; sys.path.insert(0, {repr(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))})
sys.path.insert(0, {repr(os.path.dirname(os.path.abspath(__file__)))})
import oracle
from test_gpu_pool import _k23_pool_run
err = _k23_pool_run(oracle.port(), 2, 1, n_tenants=8, dim=4096, inter=11008, n_layers=1)
assert err <= 1e-2, err
print('ok')
"""
    env = dict(os.environ, BD_DELTA="mt4")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("B,paths", [(4, "LLLL"), (16, "TTTT")])
def test_multi_plane_reference_bdelta(cuda, B, paths):
    """2- and 3-plane .bdelta files written by the reference (make_golden.py --mp) served
    through the byte LUT (1 request per tenant) and K23 (4 per tenant), against the
    reference ServingPool's logits (f32) within the bf16 tolerance."""
    d = np.load(os.path.join(GOLDEN, "mp_decode.npz"))
    arch = dict(json.loads(str(d["cfg"])))
    arch["kv_dim"] = arch["dim"]
    pool = ServingPool(arch, tensors_of(arch, d["base"]))
    for i in range(4):
        pool.register_delta(f"t{i}", os.path.join(GOLDEN, f"mp_t{i}.bdelta"))
    rids = [pool.open_request(f"t{i % 4}") for i in range(B)]
    for pos, tok in enumerate(d[f"B{B}_tokens"]):
        got = pool.decode_step([(r, int(tok), pos) for r in rids])
        assert pool.stats()["delta_paths"] == paths
        want = d[f"B{B}_logits"][pos]
        for i in range(B):
            assert rel_l2(got[i], want[i]) <= 1e-2, (pos, i, rel_l2(got[i], want[i]))
    pool.close()


def test_int8_backbone_toy_matches_port(cuda, toy, port):
    """ServingPool(QuantizedCheckpoint) (serve.cpp:99-108): the reference's own tenants on an
    RTN-int8 backbone (rtn_quantize_checkpoint with default_quantize_policy: the 7 projections),
    built on the device (ServingPool(..., int8=True) -> bd_rtn_quantize), against the port on
    rtn_dequantize of the same values; backbone residency shrinks (int8 + row scales)."""
    from paper_2402_10193_b200.serving import PROJECTIONS

    d, arch = toy
    base16 = bf16_round(d["base"])
    tens = tensors_of(arch, base16)
    names = [n for n, _, _ in tensor_shapes(arch)]
    deq = dict(tens)
    for n in names:
        if n.split(".")[-1] in PROJECTIONS:
            q, sc = port.rtn_quantize(tens[n])
            deq[n] = q.astype(np.float32) * sc[:, None]
    flat = np.concatenate([deq[n].reshape(-1) for n in names])
    tenants = [[bdelta.read(os.path.join(GOLDEN, f"toy_t{i}.bdelta"))[n] for n in names] for i in range(4)]
    dense = ServingPool(arch, tens)
    pool = ServingPool(arch, tens, int8=True)
    for i in range(4):
        pool.register_delta(f"t{i}", os.path.join(GOLDEN, f"toy_t{i}.bdelta"))
    B = 4
    rids = [pool.open_request(f"t{i}") for i in range(B)]
    kc = [np.zeros((arch["n_layers"], arch["max_seq"], arch["kv_dim"]), np.float32) for _ in range(B)]
    vc = [np.zeros_like(k) for k in kc]
    for pos, tok in enumerate(d["B4_tokens"]):
        got = pool.decode_step([(r, int(tok), pos) for r in rids])
        want = port.decode(arch, flat, tenants, list(range(B)), [int(tok)] * B, [pos] * B, kc, vc)
        for i in range(B):
            assert rel_l2(got[i], want[i]) <= 5e-3, (pos, i, rel_l2(got[i], want[i]))
    for i in range(4):
        dense.register_delta(f"t{i}", os.path.join(GOLDEN, f"toy_t{i}.bdelta"))
    # Int8Tensor::payload_bytes (int8.hpp): values + 4 B row scales instead of 4 B per weight
    proj = sum(r * c for n, r, c in tensor_shapes(arch) if n.split(".")[-1] in PROJECTIONS)
    rows = sum(r for n, r, c in tensor_shapes(arch) if n.split(".")[-1] in PROJECTIONS)
    pool.close_request(rids[0])
    for r in rids[1:]:
        pool.close_request(r)
    assert dense.resident_bytes() - pool.resident_bytes() == 4 * proj - (proj + 4 * rows)
    pool.close()
    dense.close()


def test_raw_projection_deltas_match_port(cuda, port):
    """Raw (unquantised f32) projection deltas (build_delta_file with a policy that leaves a
    projection raw; apply_delta_correction's dense branch, P:src/serve.cpp:27-35) next to
    packed ones: three tenants, one all-packed, one with raw o / down, one with raw q / gate
    (and an all-zero raw k), against the port at the bf16 tolerance. The raw groups run the
    units path + raw pass, the all-packed groups the default dispatch."""
    arch = dict(vocab=64, dim=256, n_layers=2, n_heads=2, intermediate=512, max_seq=32,
                rope_theta=10000.0, kv_dim=128)
    rng = np.random.default_rng(11)
    tens = {}
    for name, r, c in tensor_shapes(arch):
        w = rng.standard_normal((r, c)).astype(np.float32) * (1.0 if r == 1 else 0.05)
        tens[name] = bf16_round(w + (1.0 if r == 1 else 0.0))
    pool = ServingPool(arch, tens)
    ents = [_random_entries(arch, rng) for _ in range(3)]
    raw_of = {1: ("layers.0.attn_o", "layers.1.mlp_down"),
              2: ("layers.0.attn_q", "layers.1.mlp_gate", "layers.1.attn_k")}
    for t, names in raw_of.items():
        for i, (n, r, c) in enumerate(tensor_shapes(arch)):
            if n in names:
                raw = None if n == "layers.1.attn_k" else (rng.standard_normal((r, c)) * 1e-2).astype(np.float32)
                ents[t][i] = dict(name=n, kind="raw", rows=r, cols=c, raw=raw)
        assert sum(e["kind"] == "raw" and e["rows"] > 1 and "layers" in e["name"] for e in ents[t]) == len(names)
    for t, e in enumerate(ents):
        pool.register_delta_entries(f"t{t}", e)
    rids = [pool.open_request(f"t{t % 3}") for t in range(5)]
    names = [n for n, _, _ in tensor_shapes(arch)]
    port_ents = []
    for es in ents:
        pe = []
        for e in es:
            e2 = dict(e)
            if e2["kind"] == "raw":
                r2 = e2["raw"]
                e2["raw"] = (np.zeros(e2["rows"] * e2["cols"], np.float32) if r2 is None else r2.reshape(-1))
            pe.append(e2)
        port_ents.append(pe)
    # sensitivity: the same tenants with the raw projection deltas dropped
    no_raw = [[dict(e, raw=np.zeros_like(e["raw"])) if e["kind"] == "raw" and e["rows"] > 1
               and "layers" in e["name"] else e for e in es] for es in port_ents]
    flat = np.concatenate([tens[n].reshape(-1) for n in names])
    kc = [np.zeros((2, arch["max_seq"], arch["kv_dim"]), np.float32) for _ in range(5)]
    vc = [np.zeros_like(k) for k in kc]
    kc2 = [k.copy() for k in kc]
    vc2 = [v.copy() for v in vc]
    for pos in range(6):
        toks = [int(x) for x in rng.integers(0, arch["vocab"], 5)]
        got = pool.decode_step([(r, toks[i], pos) for i, r in enumerate(rids)])
        want = port.decode(arch, flat, port_ents, [i % 3 for i in range(5)], toks, [pos] * 5, kc, vc)
        want0 = port.decode(arch, flat, no_raw, [i % 3 for i in range(5)], toks, [pos] * 5, kc2, vc2)
        for i in range(5):
            # bf16 backbone activations against the f32 port: the head_dim-128 tolerance
            err = rel_l2(got[i], want[i])
            assert err <= 2e-2, (pos, i, err)
            if i % 3:  # tenants with raw projections: dropping them is well outside tolerance
                assert rel_l2(want0[i], want[i]) > 2 * 2e-2, (pos, i)
    pool.close()


def test_more_than_four_planes_match_port(cuda, port):
    """compress_stack with k > 4 (P:src/delta.cpp:57-70): planes beyond the engine's 4 per
    unit run as accumulate passes of the delta units; 6- and 9-plane projections next to
    1-plane ones, against the port (which sums every plane like apply_delta_correction)."""
    arch = dict(vocab=64, dim=256, n_layers=2, n_heads=2, intermediate=512, max_seq=32,
                rope_theta=10000.0, kv_dim=128)
    rng = np.random.default_rng(12)
    tens = {}
    for name, r, c in tensor_shapes(arch):
        w = rng.standard_normal((r, c)).astype(np.float32) * (1.0 if r == 1 else 0.05)
        tens[name] = bf16_round(w + (1.0 if r == 1 else 0.0))
    pool = ServingPool(arch, tens)
    ents = [_random_entries(arch, rng) for _ in range(2)]
    wide = {"layers.0.attn_v": 6, "layers.1.mlp_up": 9, "layers.1.mlp_down": 5}
    for i, (n, r, c) in enumerate(tensor_shapes(arch)):
        if n in wide:
            k, nb = wide[n], (r * c + 7) // 8
            ents[1][i] = dict(name=n, kind="packed", rows=r, cols=c,
                              bits=rng.integers(0, 256, (k, nb), dtype=np.uint8),
                              scales=(6e-3 * 0.9 ** np.arange(k)).astype(np.float32))
    for t, e in enumerate(ents):
        pool.register_delta_entries(f"t{t}", e)
    rids = [pool.open_request(f"t{t % 2}") for t in range(4)]
    names = [n for n, _, _ in tensor_shapes(arch)]
    port_ents = [[dict(e, raw=e["raw"].reshape(-1)) if e["kind"] == "raw" else e for e in es] for es in ents]
    # sensitivity: the same tenants with the planes beyond the 4th dropped
    cut = [[dict(e, bits=e["bits"][:4], scales=e["scales"][:4]) if e["kind"] == "packed" else e for e in es]
           for es in port_ents]
    flat = np.concatenate([tens[n].reshape(-1) for n in names])
    kc = [np.zeros((2, arch["max_seq"], arch["kv_dim"]), np.float32) for _ in range(4)]
    vc = [np.zeros_like(k) for k in kc]
    kc2, vc2 = [k.copy() for k in kc], [v.copy() for v in vc]
    worst_cut = 0.0
    for pos in range(6):
        toks = [int(x) for x in rng.integers(0, arch["vocab"], 4)]
        got = pool.decode_step([(r, toks[i], pos) for i, r in enumerate(rids)])
        want = port.decode(arch, flat, port_ents, [i % 2 for i in range(4)], toks, [pos] * 4, kc, vc)
        want4 = port.decode(arch, flat, cut, [i % 2 for i in range(4)], toks, [pos] * 4, kc2, vc2)
        for i in range(4):
            err = rel_l2(got[i], want[i])
            assert err <= 2e-2, (pos, i, err)  # bf16 activations vs the f32 port (head_dim 128)
            if i % 2:
                worst_cut = max(worst_cut, rel_l2(want4[i], want[i]))
    assert worst_cut > 2 * 2e-2, worst_cut  # dropping the extra planes is well outside tolerance
    pool.close()
