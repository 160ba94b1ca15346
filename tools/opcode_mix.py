"""Executed-instruction mix per opcode of a kernel in an ncu report (source page, SASS):
python tools/opcode_mix.py rep.ncu-rep kernel-substring [normaliser]"""
import collections
import csv
import io
import subprocess
import sys

rep, sub = sys.argv[1], sys.argv[2]
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kern, hdr = None, None
mix = collections.Counter()
seen = set()
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        kern, hdr = r[1], None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and kern and sub in kern:
        d = dict(zip(hdr, r))
        if (kern, d["Address"]) in seen:
            continue
        seen.add((kern, d["Address"]))
        src = d["Source"].strip()
        if src.startswith("@"):
            src = src.split(None, 1)[1] if " " in src else src
        op = src.split()[0] if src else "?"
        mix[op.split(".")[0]] += int(d["Instructions Executed"] or 0)
tot = sum(mix.values())
print(f"total {tot} ({tot / norm:.1f} per unit)")
for op, c in mix.most_common(40):
    print(f"{op:14s} {c / norm:8.2f}  {100 * c / tot:5.1f}%")
