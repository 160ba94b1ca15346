"""Per-instruction executed counts and stall samples of a kernel from an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass):
python tools/src_hot.py src.csv kernel-substring [positions]  -> opcode mix per position and
the stall-sampled hottest instructions."""
import collections
import csv
import sys

path, sub = sys.argv[1], sys.argv[2]
npos = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
rows, kern, hdr, done = [], None, None, set()
for r in csv.reader(open(path)):
    if r and r[0] == "Kernel Name":
        if kern and sub in kern and rows:
            done.add(kern)
        kern, hdr = r[1], None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and kern and sub in kern and kern not in done:
        rows.append(dict(zip(hdr, r)))
seen, uniq = set(), []
for d in rows:
    if d["Address"] in seen:
        continue
    seen.add(d["Address"])
    uniq.append(d)
def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
mix, smp = collections.Counter(), collections.Counter()
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
stalls = collections.Counter()
tot_s = 0
for d in uniq:
    src = d["Source"].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1]
    op = src.split()[0].split(".")[0] if src else "?"
    n = f(d["Instructions Executed"])
    mix[op] += n
    s = f(d["Warp Stall Sampling (All Samples)"])
    smp[op] += s
    tot_s += s
    for c in stall_cols:
        stalls[c] += f(d[c])
tot = sum(mix.values())
print(f"instructions {tot:.4g}  per position {tot / npos:.1f}  samples {tot_s:.0f}")
for op, n in mix.most_common(30):
    print(f"  {op:10s} {n / npos:7.2f} /pos   samples {100 * smp[op] / max(tot_s, 1):5.1f}%")
print("stalls:", ", ".join(f"{k[6:]}={100 * v / max(tot_s, 1):.1f}%" for k, v in stalls.most_common(10)))
hot = sorted(uniq, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:40]
for d in hot:
    top = sorted(stall_cols, key=lambda c: -f(d[c]))[:2]
    print(f"{d['Address']:>6s} {f(d['Warp Stall Sampling (All Samples)']) * 100 / max(tot_s, 1):5.2f}% "
          f"x{f(d['Instructions Executed']) / npos:6.2f} {d['Source'][:60]:60s} "
          + " ".join(f"{c[6:]}={f(d[c]):.0f}" for c in top))
