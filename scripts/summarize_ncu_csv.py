"""Per-(kernel, grid) summary of an ncu --csv launch list with
gpu__time_duration / dram bytes metrics: launches, mean µs, DRAM MB/launch, GB/s."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, mi, vi, ii, gi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
d = collections.defaultdict(dict)
for r in rows:
    d[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    d[r[ii]]["k"] = r[ki].split("(")[0]
    d[r[ii]]["g"] = r[gi]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for x in d.values():
    a = agg[(x["k"], x["g"])]
    a[0] += 1
    a[1] += x.get("gpu__time_duration.sum", 0)
    a[2] += x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{len(d)} launches, {tot/1e6:.3f} ms summed kernel time")
for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{100*t/tot:5.1f}%  {k[0][:42]:42s} grid {k[1]:14s} n={c:4d} avg {t/c/1e3:8.1f} us  "
          f"dram/launch {b/c/1e6:8.2f} MB  {b/t if t else 0:7.0f} GB/s")
