"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel.

    python tools/launch_summary.py launches.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
iname, imet, ival = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= ival:
        continue
    name = r[iname].split("(")[0].replace("void ", "").replace("bd::", "").replace("<unnamed>::", "")
    per[name][r[imet]] += float(r[ival].replace(",", ""))
    if r[imet] == "gpu__time_duration.sum":
        cnt[name] += 1
tot = sum(per[n]["gpu__time_duration.sum"] for n in per)
print(f"{'kernel':34s} {'launches':>8s} {'time_us':>10s} {'share':>6s} {'DRAM_MB':>9s} {'GB/s':>8s}")
for n in sorted(per, key=lambda n: -per[n]["gpu__time_duration.sum"]):
    t = per[n]["gpu__time_duration.sum"] / 1e3
    mb = (per[n]["dram__bytes_read.sum"] + per[n]["dram__bytes_write.sum"]) / 1e6
    print(f"{n[:34]:34s} {cnt[n]:8d} {t:10.1f} {per[n]['gpu__time_duration.sum'] / tot:6.3f} {mb:9.1f} "
          f"{mb / 1e3 / (t / 1e6) if t else 0:8.1f}")
print(f"total {tot / 1e3:.1f} us over {sum(cnt.values())} launches")
