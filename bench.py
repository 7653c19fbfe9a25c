"""Benchmark of the BitDelta multi-tenant decode hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload l7_stack|l7_layer|m7_stack] [--tenants T] [--batch B]

Default workload = BASELINE.json configs[2] on one GPU: the Llama-2-7B-shaped
32-layer decode layer stack, 16 distinct 1-bit deltas, batch 16 (one request
per tenant), bf16 backbone, context 128. A "step" is one decode step of the
layer stack for the whole batch (serve.cpp:240-310). Synthetic data: random
bf16 backbone; each tenant's fine-tune = base + N(0, 1e-3), compressed on the
device by K1 (untimed setup). Working set (~26 GB) >> L2 (126 MB), so no flush
is needed between steps.

value  = tokens/s over K device-timed steps (CUDA events, inputs resident).
e2e    = same through the public API with the step's activations copied from
         pinned host memory and the result copied back inside the timed region.
roofline = the dominant kernel from a profiled step (bd_pool_profile_layers:
         CUDA events on the launching stream around every kernel).
cpu_baseline = the reference library (oracle/_ref) on a bounded sample of the
         same workload, all host threads, extrapolated (rank 0, N=1 only).

N > 1 (torchrun): one process per GPU, each serving its own replica of the
workload (weak scaling, no data-path collective); time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "multi-tenant decode tokens/sec & delta-kernel HBM GB/s vs roofline, 1/2/4/8 B200"

WORKLOADS = {
    # BASELINE.json configs[2]: Llama-2-7B stack, 16 tenants, batch 16
    "l7_stack": dict(arch=dict(vocab=32000, dim=4096, kv_dim=4096, n_layers=32, n_heads=32,
                               intermediate=11008), tenants=16, batch=16, ctx=128),
    # configs[1]: one Llama-2-7B layer, 8 tenants, batch 8
    "l7_layer": dict(arch=dict(vocab=32000, dim=4096, kv_dim=4096, n_layers=1, n_heads=32,
                               intermediate=11008), tenants=8, batch=8, ctx=128),
    # configs[3]: Mistral-7B (GQA, 14336 FFN), batch 64, tenants set by --tenants
    "m7_stack": dict(arch=dict(vocab=32000, dim=4096, kv_dim=1024, n_layers=32, n_heads=32,
                               intermediate=14336), tenants=16, batch=64, ctx=128),
}
# configs[4]: Llama-2-70B (GQA, 28672 FFN), 32 tenants, batch 32; 80 layers need the 8-GPU
# row sharding (--layers N runs a shorter stack on fewer GPUs)
WORKLOADS["l70_stack"] = dict(arch=dict(vocab=32000, dim=8192, kv_dim=1024, n_layers=80, n_heads=64,
                                        intermediate=28672), tenants=32, batch=32, ctx=128)
# K1 compressor workloads (a step = one compress pass; metric GB/s of algorithmic bytes,
# (2 s_in + 1/8) B per parameter):
#   compress_f32: configs[0], one 4096 x 4096 f32 base / fine-tune pair (L2 flushed per step);
#   compress_l70: configs[4]'s compression, one tenant's 7 projection matrices of --layers
#                 Llama-2-70B layers (bf16) per step, one batched launch; N GPUs compress
#                 disjoint layer ranges (no exchange: weak scaling)
COMPRESS = {
    "compress_f32": dict(shapes=[(4096, 4096)], dtype="f32", layers=1),
    "compress_l70": dict(shapes=[(8192, 8192), (1024, 8192), (1024, 8192), (8192, 8192), (28672, 8192),
                                 (28672, 8192), (8192, 28672)], dtype="bf16", layers=2),
}
PROJ = ["attn_q", "attn_k", "attn_v", "attn_o", "mlp_gate", "mlp_up", "mlp_down"]
PROF_KINDS = ["gemm_qkv", "gemm_o", "gemm_gu", "gemm_down", "delta_qkv", "delta_o", "delta_gu",
              "delta_down", "attn", "norm", "silu", "fused_qkv", "fused_o", "fused_gu", "fused_down",
              "xq_prep"]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi needs a moment to start: wait for its first sample so the
            # timed region is covered
            t_end = time.time() + 10.0
            while not self.samples and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.02)
        except FileNotFoundError:
            self.proc = None
        return self

    def mark(self, which):
        """Bracket the timed region (wall clock); summary() keeps samples inside it."""
        setattr(self, which, time.time())

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append([time.time()] + parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        inside = [s[1:] for s in self.samples if t0 is not None and t0 <= s[0] <= (t1 or 1e30)]
        where = "timed_region"
        if not inside and self.samples:
            # region shorter than the sampling period: the sample nearest its end (under load)
            before = [s for s in self.samples if t1 is None or s[0] <= t1 + 0.1]
            inside = [(before or self.samples)[-1][1:]]
            where = "nearest_to_region"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in inside if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in inside for i in range(4) if "Active" in s[3 + i]
                          and "Not" not in s[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(inside[0][1]) if inside[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(inside), "where": where}


def algorithmic_bytes(arch, tenants, batch, wb=2):
    """wb B per backbone weight (2 bf16, 1 int8 RTN + 4 B per row scale) + P/8
    per distinct tenant (+ activations)."""
    d, kv, inter, L = arch["dim"], arch["kv_dim"], arch["intermediate"], arch["n_layers"]
    per_layer = {"qkv": (d + 2 * kv) * d, "o": d * d, "gu": 2 * inter * d, "down": d * inter}
    P = sum(per_layer.values()) * L
    rows = (d + 2 * kv + d + 2 * inter + d) * L
    base = wb * P + (4 * rows if wb == 1 else 0)
    return {"params": P, "base": base, "bits": tenants * P / 8, "per_layer": per_layer}


def kv_bytes(arch, batch, ctx):
    return 2 * 2 * batch * ctx * arch["kv_dim"] * arch["n_layers"]  # k+v, bf16


# --------------------------------------------------------------------- ours --
def build_pool(arch, n_tenants, dev, seed=0, world=1, rank=0, int8=False):
    import torch

    import paper_2402_10193_b200 as bd
    from paper_2402_10193_b200.serving import ServingPool, tensor_shapes

    g = torch.Generator(device=dev).manual_seed(seed)
    pool = ServingPool(arch, None, device=dev.index or 0, world_size=world, rank=rank)
    if world > 1:  # row-sharded pool: rank 0's NCCL id to every rank
        import torch.distributed as dist

        obj = [ServingPool.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        pool.init_comm(obj[0])
    base = {}
    for name, r, c in tensor_shapes(arch):
        if "norm" in name:
            pool.set_tensor(name, torch.ones(1, c, device=dev))
            continue
        w = (torch.randn(r, c, device=dev, generator=g) * 0.02).to(torch.bfloat16)
        if int8 and name.split(".")[-1] in PROJ:  # ServingPool(QuantizedCheckpoint): RTN on the device
            q, sc = bd.rtn_quantize(w.float())
            pool.set_tensor_i8(name, q, sc)
            del q, sc
        else:
            pool.set_tensor(name, w)
        if name.split(".")[-1] in PROJ:
            base[name] = w
        del w
    t0 = time.time()
    for t in range(n_tenants):
        ents = []
        keep = []
        for name, r, c in tensor_shapes(arch):
            if name in base:
                w = base[name]
                fine = (w.float() + torch.randn(r, c, device=dev, generator=g) * 1e-3).to(torch.bfloat16)
                bits, alpha = bd.compress_tensor(w, fine)
                del fine
                keep.append(bits)
                ents.append({"name": name, "kind": "packed", "rows": r, "cols": c, "bits": bits,
                             "scales": [alpha.item()]})
            else:  # raw entries (embed / norms / lm_head): zero delta, nothing resident
                ents.append({"name": name, "kind": "raw", "rows": r, "cols": c,
                             "raw": torch.zeros(0, device=dev)})
        pool.register_delta_entries(f"tenant{t}", _null_raw(ents))
        del keep
        torch.cuda.empty_cache()
    setup_s = time.time() - t0
    return pool, base, setup_s


def _null_raw(ents):
    """raw entries with an empty tensor are passed as NULL (all-zero raw delta)."""
    out = []
    for e in ents:
        if e["kind"] == "raw" and getattr(e["raw"], "numel", lambda: 1)() == 0:
            e = dict(e, raw=None)
        out.append(e)
    return out


def run_ours(args, rank, world, dev):
    import torch

    import paper_2402_10193_b200 as bd

    wl = WORKLOADS[args.workload]
    arch = dict(wl["arch"], rope_theta=10000.0)
    if args.layers:
        arch["n_layers"] = args.layers
    if args.inter:  # shape experiments only (not a BASELINE config)
        arch["intermediate"] = args.inter
    T = args.tenants or wl["tenants"]
    B = args.batch or wl["batch"]
    ctx = args.ctx or wl["ctx"]
    arch["max_seq"] = ctx + args.warmup + 2 * args.steps + 8
    tp = args.parallelism == "tp" and world > 1
    torch.manual_seed(0 if tp else rank)  # tp ranks must see the same activations
    # replicas: every rank its own pool and batch; tp: one row-sharded pool, same seed everywhere
    pool, _, setup_s = build_pool(arch, T, dev, seed=1234 if tp else 1234 + rank,
                                  world=world if tp else 1, rank=rank if tp else 0,
                                  int8=args.backbone == "int8")
    rids = [pool.open_request(f"tenant{b % T}") for b in range(B)]
    pos = [0] * B
    x = torch.randn(B, arch["dim"], device=dev)
    y = torch.empty_like(x)

    def reqs():
        return [(rids[b], 0, pos[b]) for b in range(B)]

    def step(xin, xout):
        pool.decode_layers(reqs(), xin, xout)
        for b in range(B):
            pos[b] += 1

    # build a real context of `ctx - 1` positions (untimed), then warm up
    for _ in range(ctx - 1):
        step(x, y)
    for _ in range(args.warmup):
        step(x, y)
    torch.cuda.synchronize()

    # ---- device-timed region: inputs resident in HBM ----
    dist_barrier(world)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = bd.launch_count()
    with ClockSampler(dev.index or 0) as clk:
        torch.cuda.synchronize()
        clk.mark("t0")
        e0.record(stream)
        for _ in range(args.steps):
            step(x, y)
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark("t1")
    dist_barrier(world)
    ms = e0.elapsed_time(e1)
    ms_max = dist_max(ms, world, dev)
    kernels_per_step = pool.stats()["kernels_last_step"]

    # ---- e2e through the public API: host activations in, host result out ----
    xh = torch.randn(B, arch["dim"]).pin_memory()
    yh = torch.empty(B, arch["dim"]).pin_memory()
    xd = torch.empty_like(x)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_steps = min(args.steps, 8)
    dist_barrier(world)
    torch.cuda.synchronize()
    e2.record(stream)
    for _ in range(e_steps):
        xd.copy_(xh, non_blocking=True)
        step(xd, y)
        yh.copy_(y, non_blocking=True)
    e3.record(stream)
    torch.cuda.synchronize()
    e2e_ms = dist_max(e2.elapsed_time(e3), world, dev) / e_steps

    # ---- profiled step (per-kernel device time, CUDA events on the launch stream) ----
    prof = profile_step(pool, reqs(), x, y)
    for b in range(B):
        pos[b] += 1
    # ---- serial profiled step: K2 and the delta kernel one after the other (the delta
    # kernel's own HBM GB/s, the metric's second half) ----
    prof_serial = profile_step(pool, reqs(), x, y, serial=True)
    for b in range(B):
        pos[b] += 1

    ms_step = ms_max / args.steps
    streams = 1 if tp else world  # independent batches in flight across the job
    tok_s = streams * B / (ms_step / 1e3)
    return dict(ms_step=ms_step, tok_s=tok_s, e2e_ms=e2e_ms, e2e_tok_s=streams * B / (e2e_ms / 1e3),
                clocks=clk.summary(), kernels_per_step=kernels_per_step, prof=prof, prof_serial=prof_serial,
                arch=arch, T=T, wb=1 if args.backbone == "int8" else 2,
                B=B, ctx=ctx, setup_s=setup_s, launches=bd.launch_count() - launches0,
                h2d=B * arch["dim"] * 4, d2h=B * arch["dim"] * 4)


def profile_step(pool, reqs, x, y, serial=False):
    import ctypes as C

    import torch

    from paper_2402_10193_b200.capi import Request, check, lib

    n = len(reqs)
    arr = (Request * n)(*[Request(r, t, p) for r, t, p in reqs])
    ms = (C.c_double * len(PROF_KINDS))()
    cnt = (C.c_uint64 * len(PROF_KINDS))()
    fn = lib().bd_pool_profile_layers_serial if serial else lib().bd_pool_profile_layers
    check(fn(pool._h, arr, n, x.data_ptr(), y.data_ptr(), ms, cnt, torch.cuda.current_stream().cuda_stream))
    return {k: {"ms": ms[i], "count": cnt[i]} for i, k in enumerate(PROF_KINDS)}


def roofline(res, hbm_peak, peak_kind):
    """Dominant kernel from the profiled step, with its algorithmic bytes per launch."""
    arch, T, B, wb = res["arch"], res["T"], res["B"], res.get("wb", 2)
    d, kv, inter = arch["dim"], arch["kv_dim"], arch["intermediate"]
    shapes = {"qkv": (d + 2 * kv, d), "o": (d, d), "gu": (2 * inter, d), "down": (d, inter)}
    algo = {}
    for g, (rows, cols) in shapes.items():
        # K2: weights once (int8: + row scales) + activations + f32 result; K3: every tenant's plane once
        w = wb * rows * cols + (4 * rows if wb == 1 else 0)
        algo[f"gemm_{g}"] = w + 2 * B * cols + 4 * B * rows
        algo[f"delta_{g}"] = T * rows * cols / 8 + 2 * B * cols + 4 * B * rows
        # fused K2+K3: the backbone tile and every tenant's plane once
        algo[f"fused_{g}"] = w + T * rows * cols / 8 + 2 * B * cols + 4 * B * rows
    prof = res["prof"]
    cand = {k: v for k, v in prof.items() if k in algo and v["count"]}
    dom = max(cand, key=lambda k: cand[k]["ms"])
    per_launch_ms = cand[dom]["ms"] / cand[dom]["count"]
    achieved = algo[dom] / (per_launch_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(dom)
    total_ms = sum(v["ms"] for v in prof.values())
    return {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
            "traffic": traffic, "algorithmic_bytes_per_launch": algo[dom],
            "avg_launch_ms": round(per_launch_ms, 5),
            "share_of_step": round(cand[dom]["ms"] / total_ms, 4) if total_ms else None}


# ------------------------------------------------------------ compression --
def run_compress(args, rank, world, dev):
    """K1 over fine-tune / base pairs resident in HBM; CUDA events around K steps."""
    import torch

    import paper_2402_10193_b200 as bd

    wl = COMPRESS[args.workload]
    f32 = wl["dtype"] == "f32"
    dt = torch.float32 if f32 else torch.bfloat16
    layers = args.layers or wl["layers"]
    g = torch.Generator(device=dev).manual_seed(77 + rank)
    pairs = []
    for _ in range(layers):
        for rows, cols in wl["shapes"]:
            base = (torch.randn(rows, cols, device=dev, generator=g) * 0.02).to(dt)
            fine = (base.float() + torch.randn(rows, cols, device=dev, generator=g) * 1e-3).to(dt)
            pairs.append((base, fine))
    params = sum(b.numel() for b, _ in pairs)
    s_in = 4 if f32 else 2
    algo = params * (2 * s_in + 1 / 8) + 4 * len(pairs)
    outs = [(torch.empty(bd.packed_size(*b.shape), dtype=torch.uint8, device=dev),
             torch.empty(1, dtype=torch.float32, device=dev)) for b, _ in pairs]
    # inputs below ~4x L2: read a 512 MB buffer between steps (a read leaves clean lines, so
    # no write-back of flush data lands inside the timed kernel)
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev) if algo < 512e6 else None

    def step():
        bd.compress_batched(pairs, outs=outs)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist_barrier(world)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = bd.launch_count()
    with ClockSampler(dev.index or 0) as clk:
        torch.cuda.synchronize()
        clk.mark("t0")
        for a, b in ev:
            if flush is not None:
                flush.sum()  # evict the inputs from L2 (read-only sweep)
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize()
        clk.mark("t1")
    launches = bd.launch_count() - launches0
    dist_barrier(world)
    ms = dist_max(sum(a.elapsed_time(b) for a, b in ev), world, dev)
    ms_step = ms / args.steps
    # e2e through the public API: host (pinned) pairs in, packed bits + alpha out, per step
    hp = [(b.cpu().pin_memory(), f.cpu().pin_memory()) for b, f in pairs]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dpairs = [(torch.empty_like(b), torch.empty_like(f)) for b, f in pairs]
    hout = [torch.empty(o.numel(), dtype=torch.uint8).pin_memory() for o, _ in outs]
    e_steps = min(args.steps, 4)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(e_steps):
        for (db, df), (hb, hf) in zip(dpairs, hp):
            db.copy_(hb, non_blocking=True)
            df.copy_(hf, non_blocking=True)
        bd.compress_batched(dpairs, outs=outs)
        for (o, _), h in zip(outs, hout):
            h.copy_(o, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = dist_max(e0.elapsed_time(e1), world, dev) / e_steps
    # parity of the measured output against a torch restatement (first matrix)
    b0, f0 = pairs[0]
    d0 = (f0.float() - b0.float()).reshape(-1)
    bits0 = outs[0][0]
    ok = bool(torch.equal(bits0, _torch_pack(d0)))
    hbm, _, kind = peaks()
    gbs = world * algo / (ms_step / 1e3) / 1e9
    line = {"metric": "delta compression (K1) GB/s of algorithmic bytes", "value": round(gbs, 1),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if f32 else "bf16",
            "data": "synthetic (base N(0,0.02), fine = base + N(0,1e-3))",
            "config": {"workload": args.workload, "matrices_per_gpu": len(pairs), "params_per_gpu": params,
                       "layers_per_gpu": layers if not f32 else None,
                       "l2": "flushed between steps (512 MB read sweep)" if flush is not None else "inputs > L2"},
            "e2e": {"value": round(world * algo / (e2e_ms / 1e3) / 1e9, 1), "unit": "GB/s",
                    "h2d_bytes_per_step": 2 * s_in * params, "d2h_bytes_per_step": sum(o.numel() for o, _ in outs)},
            "gpu_launches": launches,
            "roofline": {"kernel": "compress_kernel", "bound": "hbm", "achieved": round(algo / (ms_step / 1e3) / 1e9, 1),
                         "peak": hbm, "peak_kind": kind, "unit": "GB/s",
                         "frac": round(algo / (ms_step / 1e3) / 1e9 / hbm, 4), "traffic": None,
                         "algorithmic_bytes_per_launch": algo, "avg_launch_ms": round(ms_step, 5),
                         "share_of_step": 1.0},
            "parity_first_matrix_bits_exact": ok,
            "clocks": clk.summary()}
    return line


def _torch_pack(d):
    import torch

    v = (d > 0).to(torch.uint8)
    pad = (-v.numel()) % 8
    if pad:
        v = torch.cat([v, torch.zeros(pad, dtype=torch.uint8, device=v.device)])
    w = torch.tensor([1, 2, 4, 8, 16, 32, 64, 128], dtype=torch.int32, device=v.device)
    return (v.view(-1, 8).to(torch.int32) * w).sum(1).to(torch.uint8)


def cpu_reference_compress(budget_matrices=None):
    """The reference compress_tensor (oracle/_ref) on 4096 x 4096 f32 pairs, all host threads
    (one matrix per thread); GB/s of the same algorithmic bytes (2*4 + 1/8 B/param)."""
    import ctypes as C

    import numpy as np

    import oracle

    lib = oracle._ref_lib()
    threads = os.cpu_count() or 1
    n = budget_matrices or threads
    rows = cols = 4096
    rng = np.random.default_rng(0)
    base = [(rng.standard_normal((rows, cols), dtype=np.float32) * 0.02) for _ in range(n)]
    fine = [(b + rng.standard_normal((rows, cols), dtype=np.float32) * 1e-3).astype(np.float32) for b in base]
    bits = [np.zeros(rows * cols // 8, np.uint8) for _ in range(n)]
    fp = C.POINTER(C.c_float)
    bp = (fp * n)(*[b.ctypes.data_as(fp) for b in base])
    fpp = (fp * n)(*[f.ctypes.data_as(fp) for f in fine])
    op = (C.POINTER(C.c_uint8) * n)(*[b.ctypes.data_as(C.POINTER(C.c_uint8)) for b in bits])
    scales = np.zeros(n, np.float32)
    secs = C.c_double()
    rc = lib.dkref_time_compress(bp, fpp, C.c_uint64(n), C.c_uint64(rows), C.c_uint64(cols), C.c_uint64(threads),
                                 op, scales.ctypes.data_as(fp), C.byref(secs))
    assert rc == 0
    algo = n * rows * cols * (2 * 4 + 1 / 8)
    return {"value": round(algo / secs.value / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
            "sample": f"reference compress_tensor on {n} 4096x4096 f32 pairs, {threads} threads "
                      f"({secs.value:.2f} s)"}


def delta_kernel(res, hbm_peak, peak_kind):
    """The tenant-delta kernel on its own (serial profile: K2 and K3 one after the other):
    algorithmic bytes (every tenant plane once + activations + f32 partials) per launch /
    its average launch time, per projection group and for the dominant group."""
    arch, T, B = res["arch"], res["T"], res["B"]
    d, kv, inter = arch["dim"], arch["kv_dim"], arch["intermediate"]
    shapes = {"qkv": (d + 2 * kv, d), "o": (d, d), "gu": (2 * inter, d), "down": (d, inter)}
    prof = res["prof_serial"]
    groups = {}
    for g, (rows, cols) in shapes.items():
        k = prof.get(f"delta_{g}")
        if not k or not k["count"]:
            continue
        slices = -(-cols // 1024)
        algo = T * rows * cols / 8 + 2 * B * cols + 4 * B * rows * slices
        ms = k["ms"] / k["count"]
        groups[g] = {"gbs": round(algo / (ms / 1e3) / 1e9, 1), "avg_launch_ms": round(ms, 5),
                     "algorithmic_bytes_per_launch": algo}
    if not groups:  # K23 (base and deltas in one kernel): no separate delta kernel
        return {"kernel": "fused (K23)", "note": "deltas run inside the base GEMM kernel"}
    dom = max(groups, key=lambda g: groups[g]["avg_launch_ms"])
    return {"kernel": f"delta_{dom}", "bound": "hbm", "achieved": groups[dom]["gbs"], "peak": hbm_peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": round(groups[dom]["gbs"] / hbm_peak, 4),
            "per_group": groups, "how": "serial profiled step (K2 then K3), CUDA events on the launch stream"}


# ------------------------------------------------------------------ cpu arm --
def cpu_reference_tok_s(arch, T, B, budget_s=12.0):
    """Reference deltakit (oracle/_ref) on a bounded sample: the per-projection work
    decode_shared does for one layer (matmul_nt over the stacked batch + one
    packed_signed_accumulate per request, serve.cpp:247-254), on a row slice of
    each projection, all host threads. Extrapolated to the full stack."""
    import ctypes as C

    import numpy as np

    import oracle

    lib = oracle._ref_lib()
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(0)
    d, kv, inter, L = arch["dim"], arch["kv_dim"], arch["intermediate"], arch["n_layers"]
    shapes = [(d, d), (kv, d), (kv, d), (d, d), (inter, d), (inter, d), (d, inter)]
    # calibrate the row fraction so the sample takes ~budget_s
    frac = 1.0 / 64
    total = 0.0
    for attempt in range(2):
        total = 0.0
        for rows, cols in shapes:
            r = max(threads, int(rows * frac))
            w = (rng.standard_normal((r, cols)) * 0.02).astype(np.float32)
            x = rng.standard_normal((B, cols)).astype(np.float32)
            bits = [rng.integers(0, 256, r * cols // 8, dtype=np.uint8) for _ in range(T)]
            bp = (C.POINTER(C.c_uint8) * T)(*[b.ctypes.data_as(C.POINTER(C.c_uint8)) for b in bits])
            alpha = np.full(T, 1e-3, np.float32)
            req = np.array([b % T for b in range(B)], np.int32)
            y = np.zeros((B, r), np.float32)
            secs = C.c_double()
            rc = lib.dkref_time_multitenant_linear(
                w.ctypes.data_as(C.POINTER(C.c_float)), C.c_uint64(r), C.c_uint64(cols), bp,
                alpha.ctypes.data_as(C.POINTER(C.c_float)), req.ctypes.data_as(C.POINTER(C.c_int32)),
                x.ctypes.data_as(C.POINTER(C.c_float)), C.c_uint64(B), C.c_uint64(threads),
                y.ctypes.data_as(C.POINTER(C.c_float)), C.byref(secs))
            assert rc == 0
            total += secs.value * rows / r
        if attempt == 0:
            sample = total * frac
            if sample > 0:
                frac = min(1.0, frac * budget_s / sample / 1.5)
    step_s = total * L
    return {"value": B / step_s, "unit": "tokens/s", "cores": threads, "kind": "reference",
            "sample": f"reference matmul_nt + packed_signed_accumulate per request for the 7 projections of one "
                      f"layer on a {frac:.4f} row slice (B={B}, T={T}), {threads} threads; extrapolated x"
                      f"{1 / frac:.1f} rows x {L} layers (glue ops < 1% of reference time, excluded)",
            "step_s": step_s}


def run_reference(args):
    wl = WORKLOADS[args.workload]
    arch = dict(wl["arch"])
    T = args.tenants or wl["tenants"]
    B = args.batch or wl["batch"]
    vals = []
    res = None
    for _ in range(args.warmup):
        cpu_reference_tok_s(arch, T, B, budget_s=2.0)
    for _ in range(args.steps):
        res = cpu_reference_tok_s(arch, T, B, budget_s=8.0)
        vals.append(res["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * B / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config_of(args, arch, T, B, wl["ctx"]),
            "cpu_baseline": {k: res[k] for k in ("unit", "cores", "kind", "sample")} | {"value": v},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_of(args, arch, T, B, ctx):
    model = ("llama2-70b-shaped" if arch["dim"] == 8192 else
             "llama2-7b-shaped" if arch["kv_dim"] == arch["dim"] else "mistral-7b-shaped")
    return {"workload": args.workload, "model": model, "layers": arch["n_layers"], "tenants": T,
            "global_batch": B if args.parallelism == "tp" else B * args.gpus,
            "batch_per_gpu": B, "seq_len": ctx,
            "parallelism": (f"tp{args.gpus}" if args.parallelism == "tp" else f"replicas{args.gpus}")
            if args.gpus > 1 else "single",
            "l2": "working set > L2 (no flush needed)",
            **({"backbone": "int8 RTN (ServingPool(QuantizedCheckpoint))"} if args.backbone == "int8" else {})}


# --------------------------------------------------------------- distributed --
def dist_barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def dist_max(v, world, dev):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def spawn_ranks(n):
    """`python bench.py --gpus N` without a launcher: one process per GPU (what torchrun
    would start), rendezvous on 127.0.0.1; rank 0 prints the line."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    return max(p.wait() for p in procs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="l7_stack", choices=sorted(WORKLOADS) + sorted(COMPRESS))
    ap.add_argument("--layers", type=int, default=0, help="override the workload's layer count")
    ap.add_argument("--inter", type=int, default=0, help="override the FFN width (shape experiments)")
    ap.add_argument("--tenants", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--ctx", type=int, default=0, help="context length before timing (default: workload)")
    ap.add_argument("--parallelism", default="tp", choices=["replicas", "tp"],
                    help="N>1: one row-sharded pool over NCCL (north star, strong scaling; default) or "
                         "independent replicas (weak scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backbone", default="bf16", choices=["bf16", "int8"],
                    help="int8: ServingPool(QuantizedCheckpoint), RTN int8 projections (SURVEY §8(f)#4)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            if args.workload in COMPRESS:
                cb = cpu_reference_compress()
                print(json.dumps({"impl": "reference", "metric": "delta compression (K1) GB/s of algorithmic bytes",
                                  "value": cb["value"], "unit": "GB/s", "n_gpus": args.gpus, "steps": 1,
                                  "warmup": 0, "higher_is_better": True, "dtype": "f32", "data": "synthetic",
                                  "config": {"workload": args.workload}, "cpu_baseline": cb,
                                  "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}), flush=True)
            else:
                run_reference(args)
        return

    import torch

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    if args.workload in COMPRESS:
        line = run_compress(args, rank, world, dev)
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_reference_compress()
        if rank == 0:
            print(json.dumps(line), flush=True)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    res = run_ours(args, rank, world, dev)
    hbm, tfl, kind = peaks()
    rl = roofline(res, hbm, kind)
    byts = algorithmic_bytes(res["arch"], res["T"], res["B"], res["wb"])
    line = {"metric": METRIC, "value": round(res["tok_s"], 2), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_step"], 4),
            "higher_is_better": True,
            "scaling": "strong" if (args.parallelism == "tp" and world > 1) else "weak",
            "vs_baseline": None, "dtype": "int8+bf16" if args.backbone == "int8" else "bf16",
            "data": "synthetic (random bf16 backbone; fine = base + N(0,1e-3) compressed on device by K1)",
            "config": config_of(args, res["arch"], res["T"], res["B"], res["ctx"]),
            "e2e": {"value": round(res["e2e_tok_s"], 2), "unit": "tokens/s", "h2d_bytes_per_step": res["h2d"],
                    "d2h_bytes_per_step": res["d2h"]},
            "gpu_launches": res["kernels_per_step"] * args.steps,
            "roofline": rl,
            "delta_kernel": delta_kernel(res, hbm, kind),
            "step_roofline": {"algorithmic_bytes": byts["base"] + byts["bits"],
                              "kv_bytes": kv_bytes(res["arch"], res["B"], res["ctx"]),
                              "achieved_gbs": round((byts["base"] + byts["bits"]) / (res["ms_step"] / 1e3) / 1e9, 1),
                              "frac_of_measured_hbm": round((byts["base"] + byts["bits"]) / (res["ms_step"] / 1e3) / 1e9 / hbm, 4)},
            "clocks": res["clocks"],
            "profile_ms_per_step": {k: round(v["ms"], 4) for k, v in res["prof"].items()},
            "setup_s": round(res["setup_s"], 1)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference_tok_s(res["arch"], res["T"], res["B"])
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # the GPU number stands; say why the baseline is missing
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
