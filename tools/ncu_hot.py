"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report.

    python tools/ncu_hot.py report.ncu-rep [kernel_index] [n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
b = blocks[kidx]
hdr = b["rows"][0]
data = b["rows"][1:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
i_ex = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[i_s] or 0) for r in data)
print(b["name"], "samples", tot)
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:n]:
    st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{100 * float(r[i_s]) / tot:5.1f}% {r[0]:>6} {r[i_src][:70]:70} ex={r[i_ex]:>8} "
          + " ".join(f"{k}={v:.0f}" for v, k in st))
