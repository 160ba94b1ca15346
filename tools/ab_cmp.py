"""Compare two ab_dump.py digests: python tools/ab_cmp.py a.json b.json"""
import json
import sys

a, b = json.load(open(sys.argv[1])), json.load(open(sys.argv[2]))
bad = [k for k in a if a[k] != b.get(k)]
print(sys.argv[2], "identical" if not bad else f"DIFFER: {bad}")
