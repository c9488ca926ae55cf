"""Sum ncu per-launch metrics over the launches of one kernel family and
record per-unit traffic in a profiles/*.json file, stamped with the source
hash of the library build it was measured on (bench.py reads it back and
reports whether the build still matches).

  python tools/ncu_traffic.py --csv gpurun_out/x.csv --kernel aesc_walk_sorted \
      --units 1.2e12 --key cfg3 --out profiles/aesc_walk_traffic.json --unit-name step
Metrics expected in the CSV: dram__bytes_read.sum, dram__bytes_write.sum,
lts__t_sectors_srcunit_tex_op_read.sum (+ _op_write / _op_atom / _op_red if
present), gpu__time_duration.sum.
"""
import argparse
import csv
import json
import os
import re
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("--csv", required=True)
ap.add_argument("--kernel", required=True, help="regex on the kernel name")
ap.add_argument("--units", type=float, required=True, help="algorithmic units over all matched launches")
ap.add_argument("--unit-name", default="step")
ap.add_argument("--key", required=True)
ap.add_argument("--out", required=True)
ap.add_argument("--note", default="")
a = ap.parse_args()

scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1, "sector": 1, "": 1}
with open(a.csv) as f:
    rows = [r for r in csv.reader(line for line in f if not line.startswith("=="))]
hdr = rows[0]
ki, ii, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
pat = re.compile(a.kernel)
per = defaultdict(float)
launches = set()
for r in rows[1:]:
    if len(r) <= vi or not pat.search(r[ki]):
        continue
    launches.add(r[ii])
    per[r[mi]] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
n = max(len(launches), 1)
dram = per.get("dram__bytes_read.sum", 0.0) + per.get("dram__bytes_write.sum", 0.0)
l2 = sum(v for k, v in per.items() if k.startswith("lts__t_sectors_srcunit_tex")) * 32
red = per.get("lts__t_sectors_srcunit_tex_op_red.sum", 0.0) + per.get("lts__t_sectors_srcunit_tex_op_atom.sum", 0.0)
t = per.get("gpu__time_duration.sum", 0.0)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    srchash = open(os.path.join(root, "paper_2410_14056_b200", "libsaba_cuda.so.srchash")).read().strip()
except OSError:
    srchash = None
entry = {f"dram_bytes_per_{a.unit_name}": dram / a.units, f"l2_sector_bytes_per_{a.unit_name}": l2 / a.units,
         f"l2_reductions_per_{a.unit_name}": red / a.units, "l2_reductions_per_launch": red / n,
         "dram_bytes_per_launch": dram / n, "l2_sector_bytes_per_launch": l2 / n, "launches": len(launches),
         "units": a.units, "ncu_seconds_total": t, "kernel_regex": a.kernel, "csv": os.path.basename(a.csv),
         "srchash": srchash, "note": a.note or "ncu --clock-control none, serialised cold-ish launches"}
try:
    d = json.load(open(a.out))
except Exception:
    d = {}
d[a.key] = entry
d["_source"] = "tools/ncu_traffic.py over an ncu --metrics launch CSV; per-unit = summed over matched launches"
json.dump(d, open(a.out, "w"), indent=1)
print(json.dumps({a.key: entry}, indent=1))
