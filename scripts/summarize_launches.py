"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
tot, cnt = collections.Counter(), collections.Counter()
for r in data:
    try:
        v = float(r[vi].replace(",", "")) * scale[r[ui]]
    except (ValueError, KeyError):
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("lsb::<unnamed>::", "")
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"launches {sum(cnt.values())}, summed kernel time {T / 1e6:.2f} s over {steps:g} step(s)")
print(f"{'share':>7} {'ms/step':>10} {'launches/step':>14}  kernel")
for k, v in tot.most_common(30):
    print(f"{100 * v / T:6.2f}% {v / 1e3 / steps:10.2f} {cnt[k] / steps:14.0f}  {k[:100]}")
