"""Timing probe for the fused K2+K3 kernel through bd_multitenant_linear.

    python tools/fused_probe.py [--rows 12288 --cols 4096 --batch 16 --tenants 16]

Prints the device time per call (CUDA events, 20 reps after 3 warm-ups) and the
algorithmic HBM rate (backbone bf16 + every tenant's plane once). Knobs are
read from the environment by the library: BD_FUSED_RING, BD_FUSED_DEBUG,
BD_NO_FUSED.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_10193_b200 as bd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=12288)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--tenants", type=int, default=16)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--same-bits", action="store_true", help="all tenants share one plane (one TMA descriptor)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.manual_seed(0)
    W = (torch.randn(a.rows, a.cols, device=dev) * 0.02).to(torch.bfloat16)
    X = torch.randn(a.batch, a.cols, device=dev).to(torch.bfloat16)
    bits, alphas = [], []
    for t in range(a.tenants):
        b, al = bd.compress_tensor(W, (W.float() + 1e-3 * torch.randn_like(W.float())).to(torch.bfloat16))
        bits.append(bits[0] if (a.same_bits and bits) else b)
        alphas.append(al.item())
    rt = [b % a.tenants for b in range(a.batch)]
    for _ in range(3):
        bd.multitenant_linear(W, bits, alphas, rt, X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        bd.multitenant_linear(W, bits, alphas, rt, X)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    byts = 2 * a.rows * a.cols + a.tenants * a.rows * a.cols / 8
    print(json.dumps({"env": {k: os.environ.get(k) for k in ("BD_FUSED_RING", "BD_FUSED_DEBUG", "BD_NO_FUSED")},
                      "ms": round(ms, 4), "GBps": round(byts / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
