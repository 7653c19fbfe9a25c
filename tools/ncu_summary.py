"""Summarise an ncu report: per kernel launch, duration, DRAM bytes, throughputs, top stalls.

    python tools/ncu_summary.py report.ncu-rep [--stalls]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "MB_rd"),
    ("dram__bytes_write.sum", "MB_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:60]
        vals = []
        for m, short in METRICS:
            if m in hdr:
                v = r[hdr.index(m)]
                u = units[hdr.index(m)]
                try:
                    f = float(v)
                    if short.startswith("MB") and u.lower() == "gbyte":
                        f *= 1000
                    if short.startswith("MB") and u.lower() == "kbyte":
                        f /= 1000
                    if short == "us" and u == "ms":
                        f *= 1000
                    vals.append(f"{short}={f:.1f}")
                except ValueError:
                    vals.append(f"{short}={v}")
        print(name, " ".join(vals))
        if "--stalls" in sys.argv:
            st = []
            for i, h in enumerate(hdr):
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                    try:
                        st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main()
