"""Per-kernel share of a step from an ncu launch list (--metrics gpu__time_duration.sum --csv):
python tools/launch_summary.py gpurun_out/r02_launches.csv "<command note>" > profiles/r02_launches.md"""
import collections
import csv
import re
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
hdr, agg = None, collections.OrderedDict()
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    m = re.search(r"(\w+_kernel)(<[^>]*>)?", d["Kernel Name"])
    key = m.group(1) if m else d["Kernel Name"][:40]
    if key == "sweep_kernel":
        ta = m.group(2).replace("(int)", "").replace("(bool)", "").strip("<>").split(",")
        key = "sweep_bwd_wta" if ta[2].strip() in ("1", "true") else "sweep_fwd"
    v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d.get("Metric Unit", ""), 1.0)
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
print("# kernel launch list (ncu gpu__time_duration, --clock-control none)\n")
print(sys.argv[2] if len(sys.argv) > 2 else "")
print("\n| kernel | launches | total us | us/launch | share |\n|---|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {n} | {t:.1f} | {t / n:.1f} | {100 * t / tot:.1f}% |")
