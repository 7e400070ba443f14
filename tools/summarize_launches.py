"""Summarise an ncu --csv launch list by kernel: device time share, average
time, DRAM bytes per launch and achieved DRAM GB/s (metrics
gpu__time_duration.sum [, dram__bytes_read.sum, dram__bytes_write.sum]).
Optional second argument: skip the first N launches (warm-up); --json OUT
writes per-kernel DRAM bytes per launch (bench.py reads profiles/traffic.json)."""
import json
import collections
import csv
import sys

UNITS = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "s": 1e6, "second": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}
args = [a for a in sys.argv[1:]]
jout = None
if "--json" in args:
    jout = args[args.index("--json") + 1]
    del args[args.index("--json"):args.index("--json") + 2]
rows = list(csv.reader(open(args[0])))
skip = int(args[1]) if len(args) > 1 else 0
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ki, ii, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "ID", "Metric Name", "Metric Value",
                                             "Metric Unit"))
agg = collections.defaultdict(lambda: collections.defaultdict(float))
launches = collections.defaultdict(set)
for r in rows[hi + 1:]:
    if len(r) <= vi or int(r[ii]) < skip:
        continue
    v = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
    name = r[ki].split("(")[0][:60]
    agg[name][r[mi]] += v
    launches[name].add(r[ii])
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"total {tot / 1e3:.3f} ms over {sum(len(v) for v in launches.values())} launches")
for name, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    t, n = a["gpu__time_duration.sum"], len(launches[name])
    b = a.get("dram__bytes_read.sum", 0.0) + a.get("dram__bytes_write.sum", 0.0)
    print(f"{100 * t / tot:6.2f}%  {t / 1e3:9.3f} ms  n={n:5d}  avg={t / n:9.1f} us  "
          f"dram/launch={b / n / 1e6:8.1f} MB  {b / t / 1e3 if t else 0:6.0f} GB/s  {name}")

if jout:
    ker = {}
    for name, a in agg.items():  # template instantiations aggregate under the base name
        short = name.split("::")[-1].split("<")[0].strip()
        k = ker.setdefault(short, {"launches": 0, "us": 0.0, "bytes": 0.0})
        k["launches"] += len(launches[name])
        k["us"] += a["gpu__time_duration.sum"]
        k["bytes"] += a.get("dram__bytes_read.sum", 0.0) + a.get("dram__bytes_write.sum", 0.0)
    ker = {s: {"launches": k["launches"], "avg_us": k["us"] / k["launches"],
               "dram_bytes_per_launch": k["bytes"] / k["launches"]} for s, k in ker.items()}
    json.dump({"source": args[0], "kernels": ker}, open(jout, "w"), indent=1)
