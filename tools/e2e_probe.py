"""Where the e2e step (host activations in, host result out) loses against the device-resident
step on the default workload (experiments): per-step ms of several loop variants."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

wl = bench.WORKLOADS["l7_stack"]
arch = dict(wl["arch"], rope_theta=10000.0)
T, B, ctx = wl["tenants"], wl["batch"], wl["ctx"]
arch["max_seq"] = ctx + 400
dev = torch.device("cuda:0")
pool, _, _ = bench.build_pool(arch, T, dev, seed=1234)
rids = [pool.open_request(f"tenant{b % T}") for b in range(B)]
pos = [0] * B
x = torch.randn(B, arch["dim"], device=dev)
y = torch.empty_like(x)


def step(xin, xout):
    pool.decode_layers([(rids[b], 0, pos[b]) for b in range(B)], xin, xout)
    for b in range(B):
        pos[b] += 1


for _ in range(ctx + 5):
    step(x, y)
torch.cuda.synchronize()
xh = torch.randn(B, arch["dim"]).pin_memory()
yh = torch.empty(B, arch["dim"]).pin_memory()
xd = torch.empty_like(x)
s = torch.cuda.current_stream()


def timed(n, body):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        body()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


res = {}
for n in (8, 30):
    res[f"resident_{n}"] = timed(n, lambda: step(x, y))
    res[f"other_input_{n}"] = timed(n, lambda: step(xd, y))
    res[f"h2d_{n}"] = timed(n, lambda: (xd.copy_(xh, non_blocking=True), step(xd, y)))
    res[f"h2d_d2h_{n}"] = timed(n, lambda: (xd.copy_(xh, non_blocking=True), step(xd, y), yh.copy_(y, non_blocking=True)))
for k, v in res.items():
    print(f"{k:16s} {v:.4f} ms/step")
