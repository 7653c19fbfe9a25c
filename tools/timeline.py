"""Device timeline of one decode step (bd_trace_enable): per launch of the K2/K3/glue
kernels, when its CTAs entered, passed griddepcontrol.wait and exited (%globaltimer).

    python tools/timeline.py [--workload l7_stack] [--out gpurun_out/timeline.txt]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KIND = {1: "lut", 2: "k2", 3: "norm", 4: "attn", 5: "silu"}
REC = np.dtype([("kind", "<u4"), ("cta", "<u4"), ("smid", "<u4"), ("pad", "<u4"),
                ("t_entry", "<u8"), ("t_wait", "<u8"), ("t_end", "<u8")])


def launches(recs):
    out = []
    for k in sorted(set(recs["kind"].tolist())):
        r = np.sort(recs[recs["kind"] == k], order="t_entry")
        cur, seen = [], set()
        for x in r:
            if x["cta"] in seen:
                out.append((k, np.array(cur, dtype=REC)))
                cur, seen = [], set()
            cur.append(x)
            seen.add(int(x["cta"]))
        if cur:
            out.append((k, np.array(cur, dtype=REC)))
    out.sort(key=lambda t: int(t[1]["t_entry"].min()))
    return out


def main():
    import torch

    import bench
    import paper_2402_10193_b200 as bd  # noqa: F401
    from paper_2402_10193_b200.capi import check, lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="l7_stack")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "timeline.txt"))
    ap.add_argument("--tenants", type=int, default=0)
    args = ap.parse_args()
    wl = bench.WORKLOADS[args.workload]
    arch = dict(wl["arch"], rope_theta=10000.0)
    T, B, ctx = args.tenants or wl["tenants"], wl["batch"], wl["ctx"]
    arch["max_seq"] = ctx + 16
    dev = torch.device("cuda:0")
    pool, _, _ = bench.build_pool(arch, T, dev, seed=1234)
    rids = [pool.open_request(f"tenant{b % T}") for b in range(B)]
    pos = [0] * B
    x = torch.randn(B, arch["dim"], device=dev)
    y = torch.empty_like(x)

    def step():
        pool.decode_layers([(rids[b], 0, pos[b]) for b in range(B)], x, y)
        for b in range(B):
            pos[b] += 1

    for _ in range(ctx + 3):
        step()
    torch.cuda.synchronize()
    cap = 1 << 20
    check(lib().bd_trace_enable(cap))
    step()
    torch.cuda.synchronize()
    buf = np.zeros(cap, dtype=REC)
    n = C.c_uint32()
    check(lib().bd_trace_read(buf.ctypes.data, cap, C.byref(n)))
    check(lib().bd_trace_enable(0))
    recs = buf[: n.value]
    L = launches(recs)
    t0 = int(recs["t_entry"].min())
    lines = [f"# {args.workload}: {len(L)} launches, {n.value} CTA records; times in us from the first entry",
             "# kind  ctas  entry0  wait_med  end_med  end_max  (dur=end_max-entry0, tail=end_max-end_med, gap=entry0-prev_end_max)"]
    prev_end = None
    agg = {}
    for k, r in L:
        e0 = (int(r["t_entry"].min()) - t0) / 1e3
        wm = (float(np.median(r["t_wait"].astype(np.float64))) - t0) / 1e3
        em = (float(np.median(r["t_end"].astype(np.float64))) - t0) / 1e3
        ex = (int(r["t_end"].max()) - t0) / 1e3
        gap = "" if prev_end is None else f" gap={e0 - prev_end:7.2f}"
        lines.append(f"{KIND[k]:5s} {len(r):5d} {e0:9.2f} {wm:9.2f} {em:9.2f} {ex:9.2f} dur={ex - e0:7.2f} "
                     f"tail={ex - em:6.2f}{gap}")
        a = agg.setdefault(KIND[k], [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += ex - e0
        a[2] += ex - em
        a[3] += wm - e0
        prev_end = ex if prev_end is None else max(prev_end, ex)
    span = (int(recs["t_end"].max()) - t0) / 1e3
    lines.append(f"# step span {span:.1f} us")
    for k, (c, d, t, w) in agg.items():
        lines.append(f"# {k:5s} launches={c:4d} sum_dur={d:8.1f} us  mean_dur={d / c:6.2f}  mean_tail={t / c:5.2f}  "
                     f"mean_entry_to_wait={w / c:5.2f}")
    # critical-path view: time where no K2/K3 CTA is running
    iv = sorted(((int(x["t_entry"]), int(x["t_end"])) for x in recs if x["kind"] in (1, 2)))
    busy, cs, ce = 0, None, None
    for s_, e_ in iv:
        if cs is None or s_ > ce:
            if cs is not None:
                busy += ce - cs
            cs, ce = s_, e_
        else:
            ce = max(ce, e_)
    if cs is not None:
        busy += ce - cs
    lines.append(f"# time with at least one K2/K3 CTA alive: {busy / 1e3:.1f} us of {span:.1f}")
    # LUT tail anatomy: for the first launches of each LUT shape, end time vs the number of
    # K2 CTAs that ran on the same SM during the LUT, and vs the SM index (die)
    k2 = recs[recs["kind"] == 2]
    for li, (k, r) in enumerate(L[:12]):
        if k != 1:
            continue
        t_lo, t_hi = int(r["t_entry"].min()), int(r["t_end"].max())
        ov = k2[(k2["t_end"] > t_lo) & (k2["t_entry"] < t_hi)]
        per_sm = np.bincount(ov["smid"].astype(np.int64), minlength=160)
        ends = (r["t_end"].astype(np.float64) - float(r["t_end"].min())) / 1e3
        nk = per_sm[r["smid"].astype(np.int64)]
        die = (r["smid"] >= 74).astype(int)
        lines.append(f"# LUT launch {li}: end spread {ends.max():.2f} us; mean end by K2-CTAs-on-SM: " +
                     " ".join(f"{c}:{ends[nk == c].mean():.2f}(n={int((nk == c).sum())})" for c in sorted(set(nk.tolist()))) +
                     f"; by smid>=74: {ends[die == 0].mean():.2f}/{ends[die == 1].mean():.2f}; "
                     f"corr(end, cta)={np.corrcoef(ends, r['cta'].astype(np.float64))[0, 1]:.2f}")
    # per-SM lateness of the LUT launches: is the same SM late in every launch?
    lut = [r for k, r in L if k == 1]
    if len(lut) >= 8:
        M = np.full((len(lut), 160), np.nan)
        for i, r in enumerate(lut):
            e = (r["t_end"].astype(np.float64) - np.median(r["t_end"].astype(np.float64))) / 1e3
            M[i, r["smid"].astype(np.int64)] = e
        half = len(lut) // 2
        a_ = np.nanmean(M[:half], axis=0)
        b_ = np.nanmean(M[half:], axis=0)
        ok = ~np.isnan(a_) & ~np.isnan(b_)
        lines.append(f"# LUT per-SM lateness: corr(first half of launches, second half) = "
                     f"{np.corrcoef(a_[ok], b_[ok])[0, 1]:.2f}; per-SM mean lateness std {np.nanstd(np.nanmean(M, axis=0)):.2f} us, "
                     f"per-launch std {np.nanmean(np.nanstd(M, axis=1)):.2f} us")
        np.save(os.path.join(os.path.dirname(args.out), "lut_sm_lateness.npy"), M)
    txt = "\n".join(lines)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    open(args.out, "w").write(txt + "\n")
    print("\n".join(lines[:2] + lines[-8:]))


if __name__ == "__main__":
    main()
