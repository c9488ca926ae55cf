"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

tot, cnt = defaultdict(float), defaultdict(int)
with open(sys.argv[1]) as f:
    rows = [r for r in csv.reader(line for line in f if not line.startswith("=="))]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    full = r[ki].replace("void ", "").replace("saba_cu::<unnamed>::", "")
    base = full.split("(")[0]
    name = base.split("<")[0] + ("<" + base.split("<", 1)[1] if "<" in base and "cub::" not in base else "")
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{k[:70]:70s} {cnt[k]:8d} {v:10.3f} {100*v/T:6.1f}%")
print(f"{'total':70s} {sum(cnt.values()):8d} {T:10.3f}")
