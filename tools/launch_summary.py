"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.

usage: launch_summary.py LIST.csv [START_KERNEL N]: with START_KERNEL, only the launches from
the N-th launch whose name contains START_KERNEL up to the (N+1)-th are counted (one
micro-batch of tools/profile_micro.py: START_KERNEL = embed_fwd_kernel, N = 2)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
data = [d for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
if len(sys.argv) > 3:
    key, nth = sys.argv[2], int(sys.argv[3])
    marks = [i for i, d in enumerate(data) if key in d["Kernel Name"]]
    data = data[marks[nth - 1]: marks[nth] if len(marks) > nth else len(data)]
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"n": 1e-3, "u": 1.0, "m": 1e3}
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", d["Kernel Name"])
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"].strip()[:1], 1e-3)
tot = sum(v[1] for v in agg.values())
print(f"{len(data)} launches, {tot / 1e3:.2f} ms total (cold-cache, serialised)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1] / 1e3:9.3f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:4d}  avg {v[1] / v[0]:9.1f} us  {k[:100]}")
