"""Multi-GPU dataflow of the pool (output-row sharding + per-layer all-gathers,
csrc/pool.cu run_layers / paper_2402_10193_b200.sharding) validated on CPU with
world_size 2 over gloo: every rank computes its row shard of every projection
and of each tenant's packed planes (sliced as byte ranges of the reference
layout) with the oracle's primitives, exchanges ctx / o / act / down slices by
all-gather, and the result must equal the unsharded oracle decode bit for bit
(each output row is the same dot product in the same order)."""
import json
import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _toy():
    import sys

    sys.path.insert(0, ROOT)
    from paper_2402_10193_b200 import bdelta
    from paper_2402_10193_b200.serving import tensor_shapes

    d = np.load(os.path.join(GOLDEN, "toy_decode.npz"))
    cfg = json.loads(str(d["cfg"]))
    arch = dict(cfg, kv_dim=cfg["dim"])
    names = [n for n, _, _ in tensor_shapes(arch)]
    base, off = {}, 0
    for n, r, c in tensor_shapes(arch):
        base[n] = d["base"][off:off + r * c].reshape(r, c)
        off += r * c
    tenants = [bdelta.read(os.path.join(GOLDEN, f"toy_t{i}.bdelta")) for i in range(4)]
    return arch, names, d["base"], base, tenants


def _sharded_stack(rank, world, arch, base, tenants, req_tenant, xs, port, gather):
    """Rank-local layer stack mirroring PoolImpl::run_layers for world > 1."""
    from paper_2402_10193_b200 import sharding

    f32 = np.float32
    dim, kv, inter, H = arch["dim"], arch["kv_dim"], arch["intermediate"], arch["n_heads"]
    hd = dim // H
    B = len(req_tenant)
    L = arch["n_layers"]
    q0, ql = sharding.local_rows(arch, "attn_q", world, rank)
    k0, kl = sharding.local_rows(arch, "attn_k", world, rank)
    heads_l, kvh_l = ql // hd, kl // hd
    group = heads_l // kvh_l
    inv_sqrt_hd = f32(1.0) / np.sqrt(f32(hd))
    kc = np.zeros((B, L, arch["max_seq"], kl), f32)
    vc = np.zeros_like(kc)

    def linear(role, l, x):
        name = f"layers.{l}.{role}"
        r0, nr = sharding.local_rows(arch, role, world, rank)
        W = base[name][r0:r0 + nr]
        y = port.matmul_nt(x, W)  # backbone_linear_nt on the shard
        for b in range(B):
            e = tenants[req_tenant[b]][name]
            cols = e["cols"]
            lo, hi = sharding.plane_bytes(r0, nr, cols)
            for k in range(e["planes"]):
                tmp = port.packed_signed_accumulate(e["bits"][k][lo:hi], nr, cols, x[b])
                y[b] = y[b] + f32(e["scales"][k]) * tmp  # apply_delta_correction (serve.cpp:22-26)
        return y

    def norm(x, l, which):
        out = np.zeros_like(x)
        for b in range(B):
            t = tenants[req_tenant[b]][f"layers.{l}.{which}"]
            w = (base[f"layers.{l}.{which}"][0] + t["raw"][0]).astype(f32)
            out[b] = port.rmsnorm_row(x[b], w)
        return out

    outs = []
    for step, x_in in enumerate(xs):
        x = x_in.copy()
        pos = step
        for l in range(L):
            xn = norm(x, l, "norm1")
            q, k, v = linear("attn_q", l, xn), linear("attn_k", l, xn), linear("attn_v", l, xn)
            ctx = np.zeros((B, ql), f32)
            for b in range(B):
                for h in range(heads_l):
                    q[b, h * hd:(h + 1) * hd] = port.rope_row(q[b, h * hd:(h + 1) * hd], pos, arch["rope_theta"])
                for h in range(kvh_l):
                    k[b, h * hd:(h + 1) * hd] = port.rope_row(k[b, h * hd:(h + 1) * hd], pos, arch["rope_theta"])
                kc[b, l, pos] = k[b]
                vc[b, l, pos] = v[b]
                n_ctx = pos + 1
                for h in range(heads_l):
                    qh = q[b, h * hd:(h + 1) * hd]
                    kh = h // group
                    scores = np.zeros(n_ctx, f32)
                    for j in range(n_ctx):
                        acc = f32(0.0)
                        kj = kc[b, l, j, kh * hd:(kh + 1) * hd]
                        for d in range(hd):
                            acc = f32(acc + f32(qh[d] * kj[d]))
                        scores[j] = f32(acc * inv_sqrt_hd)
                    scores = port.softmax_row(scores)
                    ch = np.zeros(hd, f32)
                    for j in range(n_ctx):
                        vj = vc[b, l, j, kh * hd:(kh + 1) * hd]
                        for d in range(hd):
                            ch[d] = f32(ch[d] + f32(scores[j] * vj[d]))
                    ctx[b, h * hd:(h + 1) * hd] = ch
            ctx_full = gather(ctx)  # exchange 1: attention context
            o_full = gather(linear("attn_o", l, ctx_full))  # exchange 2: o-projection rows
            x = (x + o_full).astype(f32)
            xn = norm(x, l, "norm2")
            g, u = linear("mlp_gate", l, xn), linear("mlp_up", l, xn)
            act = np.zeros_like(g)
            for b in range(B):
                for i in range(g.shape[1]):
                    act[b, i] = f32(port.lib.bdo_silu(float(g[b, i])) * u[b, i])
            act_full = gather(act)  # exchange 3: MLP activation
            down_full = gather(linear("mlp_down", l, act_full))  # exchange 4: down rows
            x = (x + down_full).astype(f32)
        outs.append(x)
    return outs


def _worker(rank, world, port_num, q):
    import torch
    import torch.distributed as dist

    import oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_num}", rank=rank, world_size=world)
    try:
        arch, names, flat, base, tenants = _toy()
        port = oracle.port()
        req_tenant = [0, 1, 2, 3]
        rng = np.random.default_rng(7)
        xs = [rng.standard_normal((4, arch["dim"])).astype(np.float32) for _ in range(3)]

        def gather(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            return np.concatenate([p.numpy() for p in parts], axis=1)

        outs = _sharded_stack(rank, world, arch, base, tenants, req_tenant, xs, port, gather)
        q.put((rank, [o.tolist() for o in outs]))
    finally:
        dist.destroy_process_group()


def test_row_sharded_stack_equals_unsharded_oracle():
    import torch.multiprocessing as mp

    import oracle
    from paper_2402_10193_b200.serving import tensor_shapes

    arch, names, flat, base, tenants = _toy()
    port = oracle.port()
    ents = [[t[n] for n in names] for t in tenants]
    rng = np.random.default_rng(7)
    xs = [rng.standard_normal((4, arch["dim"])).astype(np.float32) for _ in range(3)]
    kc = [np.zeros((arch["n_layers"], arch["max_seq"], arch["kv_dim"]), np.float32) for _ in range(4)]
    vc = [np.zeros_like(k) for k in kc]
    want = [port.decode(arch, flat, ents, [0, 1, 2, 3], None, [s] * 4, kc, vc, layers_only=True, x_in=x)
            for s, x in enumerate(xs)]

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_num = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port_num, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(WORLD):
        for s in range(len(xs)):
            got = np.array(results[r][s], np.float32)
            assert np.array_equal(got, want[s]), (r, s, np.abs(got - want[s]).max())


def test_plane_byte_ranges_partition_the_plane():
    """Row shards of a packed plane are disjoint contiguous byte ranges covering it."""
    from paper_2402_10193_b200 import sharding

    arch = {"dim": 4096, "kv_dim": 1024, "n_heads": 32, "intermediate": 14336}
    for world in (1, 2, 4, 8):
        sharding.check(arch, world)
        for role in sharding.PROJ:
            cols = arch["intermediate"] if role == "mlp_down" else arch["dim"]
            covered = []
            for r in range(world):
                r0, nr = sharding.local_rows(arch, role, world, r)
                covered.append(sharding.plane_bytes(r0, nr, cols))
            assert covered[0][0] == 0
            assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
            rows = sharding.local_rows(arch, role, 1, 0)[1]
            assert covered[-1][1] == rows * cols // 8
