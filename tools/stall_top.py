"""Top stall sites of a kernel in an ncu report: python tools/stall_top.py rep.ncu-rep [N]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kern, hdr, data = None, None, collections.defaultdict(list)
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        kern, hdr = r[1], None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and kern:
        data[kern].append(dict(zip(hdr, r)))
for k, v in data.items():
    seen, u = set(), []
    for d in v:
        if d["Address"] not in seen:
            seen.add(d["Address"])
            u.append(d)
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    agg = collections.Counter()
    for d in u:
        for c in cols:
            agg[c] += int(d[c] or 0)
    S = sum(agg.values()) or 1
    tot = sum(int(d["Instructions Executed"] or 0) for d in u)
    allsamp = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in u)
    print("==", k[:100], "instructions", tot, "samples", allsamp)
    print("   " + ", ".join(f"{c[6:]}={v / S * 100:.1f}%" for c, v in agg.most_common(10)))
    for d in sorted(u, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:N]:
        reason = max(cols, key=lambda c: int(d[c] or 0))
        print(f"   {int(d['Warp Stall Sampling (All Samples)']):6d} {reason[6:]:14s} "
              f"{d['Source'].strip()[:60]:60s} {d['Instructions Executed']}")
